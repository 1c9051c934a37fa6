"""TEST INFRASTRUCTURE ONLY: CPU oracle for parity checks (see gpt_oracle.py).
Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline leg; never from the product package."""
