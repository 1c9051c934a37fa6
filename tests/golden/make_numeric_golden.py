"""Generate the numeric golden fixtures at the benchmarked widths with the
float64 CPU oracle (run once in the build container; the GPU box only reads
the committed ``numeric_*.pt``).  See ``numeric.py`` for what is stored.

Each case (``numeric.case_specs``): the reduced-depth model at full width,
BitPipe with the F2 paper-gate order and the cost-balanced partition, seeded
parameters (``init_params(cfg, 7, perturb=True)``) and tokens
(``synthetic_batch(cfg, N, seed=11)``), AdamW lr 1e-3 wd 0.01.  The oracle
executes the reference-format dump of that order with message passing
(SPEC run_schedule_numeric); schedule independence of that executor is
tested separately (tests/test_oracle.py, tests/test_oracle_pinning.py).

Usage:  python tests/golden/make_numeric_golden.py [case ...]   (~1-5 min per case)
"""
from __future__ import annotations

import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.gpt_oracle import OracleConfig, run_schedule_numeric  # noqa: E402
from paper_2410_19367_b200 import schedule as ps  # noqa: E402
from paper_2410_19367_b200.model import OptimConfig, init_params, stage_partition, synthetic_batch  # noqa: E402
from tests.golden import numeric  # noqa: E402


def make(name):
    cfg, sched, counts = numeric.case(name)
    opt = OptimConfig(lr=numeric.LR, weight_decay=numeric.WD)
    params = init_params(cfg, numeric.PARAM_SEED, perturb=True)
    tok, tgt = synthetic_batch(cfg, sched.N, seed=numeric.DATA_SEED)
    oc = OracleConfig(cfg.layers, cfg.hidden, cfg.heads, cfg.seq, cfg.vocab, cfg.micro_batch, cfg.causal,
                      cfg.ln_eps, opt.lr, opt.beta1, opt.beta2, opt.eps, opt.weight_decay)
    hbs = [p.halfblocks for p in stage_partition(cfg, sched.num_stages, counts)]
    t0 = time.time()
    ref = run_schedule_numeric(oc, ps.dump_schedule(sched), params, tok, tgt, halfblocks=hbs)
    dt = time.time() - t0
    upd = {k: ref.params[k] - params[k].double() for k in params}
    fx = {"case": name, "config": cfg.__dict__ | {}, "D": sched.D, "N": sched.N,
          "policy": list(ps.paper_policy(sched.D).__dict__.values()), "partition": counts,
          "optim": opt.__dict__ | {}, "param_seed": numeric.PARAM_SEED, "data_seed": numeric.DATA_SEED,
          "schedule_sha": __import__("hashlib").sha256(ps.dump_schedule(sched).encode()).hexdigest(),
          "losses": ref.losses.clone(), "grads": numeric.summarize(ref.grads), "update": numeric.summarize(upd),
          "oracle_seconds": dt, "threads": torch.get_num_threads()}
    torch.save(fx, numeric.path(name))
    print(f"{name}: losses {ref.losses.tolist()} ({dt:.0f} s) -> {numeric.path(name)}")


if __name__ == "__main__":
    torch.set_num_threads(os.cpu_count() or 1)
    for name in sys.argv[1:] or list(numeric.case_specs()):
        make(name)
