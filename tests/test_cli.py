"""The pipesched-compatible CLI (the reference declares the
console script but ships no cli.py, pkg/pyproject.toml:19-20)."""
import hashlib
import json

import pytest

from paper_2410_19367_b200.cli import main

GOLD_BITPIPE_D4_N8 = "28b3f28155b2cb85b510a41d0ef59c4b7a01b5cd2c54c502ce72e439f93108c9"


def run(capsys, *argv):
    rc = main(list(argv))
    out = capsys.readouterr()
    return rc, out.out, out.err


def test_plan_is_byte_equal_to_reference_dump(capsys):
    rc, out, _ = run(capsys, "plan", "--approach", "bitpipe", "--D", "4", "--N", "8")
    assert rc == 0 and hashlib.sha256(out.encode()).hexdigest() == GOLD_BITPIPE_D4_N8


def test_plan_writes_files(tmp_path, capsys):
    rc, _, _ = run(capsys, "plan", "--approach", "bitpipe", "--approach", "chimera", "--D", "4", "--N", "8",
                   "--out", str(tmp_path))
    assert rc == 0
    assert sorted(p.name for p in tmp_path.iterdir()) == ["bitpipe_D4_N8.json", "chimera_D4_N8.json"]


@pytest.mark.parametrize("argv,code", [
    (["plan", "--approach", "nope"], 1),                           # unknown approach: usage error
    (["plan"], 1),                                                 # empty approach list
    (["plan", "--bogus"], 1),                                      # bad flag
    (["plan", "--approach", "bitpipe", "--D", "3", "--N", "6"], 2),  # OddDeviceCount: domain error
    (["plan", "--approach", "bitpipe", "--D", "4", "--N", "6"], 2),  # InvalidChunking
    (["plan", "--approach", "bitpipe", "--D", "6", "--N", "12", "--order", "paper"], 1),  # no F2 gate for D=6
])
def test_exit_codes(argv, code, capsys):
    rc, _, _ = run(capsys, *argv)
    assert rc == code


def test_compare_rows(capsys):
    rc, out, _ = run(capsys, "compare", "--approach", "bitpipe", "--D", "8", "--N", "16", "--format", "json")
    rows = json.loads(out)
    assert rc == 0 and rows[0]["bubble_analytic"] == "1/9" and rows[0]["bubble_sim"] == "5/13"
    rc, out, _ = run(capsys, "compare", "--approach", "bitpipe", "--D", "8", "--N", "16", "--order", "paper",
                     "--format", "json")
    assert json.loads(out)[0]["bubble_sim"] == "1/9"  # F2 order reaches the analytic bubble


def test_simulate_timeline_and_svg(tmp_path, capsys):
    rc, out, _ = run(capsys, "simulate", "--approach", "bitpipe", "--D", "4", "--N", "8")
    tl = json.loads(out)
    assert rc == 0 and len(tl["tasks"]) == 4 * 4 * 8 and tl["makespan"] == "36"
    rc, _, _ = run(capsys, "simulate", "--approach", "bitpipe", "--D", "8", "--N", "16", "--model", "gpt-1.3b",
                   "--partition", "balanced", "--format", "svg", "--out", str(tmp_path))
    svg = (tmp_path / "bitpipe_D8_N16.svg").read_text()
    assert rc == 0 and svg.startswith("<svg") and svg.count("<rect") == 8 * 4 * 16


def test_search_best_row(capsys):
    rc, out, _ = run(capsys, "search", "--approach", "bitpipe", "--approach", "1f1b", "--D", "8", "--N", "16",
                     "--order", "both", "--format", "json")
    rows = json.loads(out)
    assert rc == 0 and rows[-1]["approach"] == "BEST:bitpipe" and rows[-1]["order"] == "paper"


def test_render_ascii(capsys):
    rc, out, _ = run(capsys, "render", "--approach", "bitpipe", "--D", "4", "--N", "4")
    lines = out.strip().splitlines()
    assert rc == 0 and len(lines) == 4 and lines[0].startswith("dev0: F1d0")


def test_verify_structure(capsys):
    rc, out, _ = run(capsys, "verify", "--approach", "bitpipe", "--approach", "bitpipe-ef", "--approach", "chimera",
                     "--D", "2", "--D", "4", "--D", "8")
    assert rc == 0 and out.count("ok") == 9 and "FAIL" not in out


@pytest.mark.gpu
def test_verify_gpu_schedule_independence(capsys):
    rc, out, _ = run(capsys, "verify", "--gpu", "--approach", "bitpipe", "--approach", "chimera", "--D", "2",
                     "--D", "4")
    assert rc == 0 and out.count("ok   gpu") == 4, out


def test_measure_needs_gpu_on_cpu_box(capsys):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    rc, _, err = run(capsys, "measure", "--approach", "bitpipe", "--D", "2", "--N", "4")
    assert rc == 2 and "CUDA" in err


@pytest.mark.gpu
def test_measure_timeline(capsys):
    rc, out, _ = run(capsys, "measure", "--approach", "bitpipe", "--D", "4", "--N", "8", "--model", "tiny",
                     "--dtype", "fp32")
    tl = json.loads(out)
    assert rc == 0 and len(tl["tasks"]) == 4 * 4 * 8 and float(tl["makespan"]) > 0
    assert all(float(t["end"]) >= float(t["start"]) for t in tl["tasks"])


def test_search_order_with_memory_cap(capsys):
    rc, out, _ = run(capsys, "compare", "--approach", "bitpipe", "--D", "8", "--N", "16", "--order", "search",
                     "--max-peak", "8", "--format", "json")
    rows = json.loads(out)
    assert rc == 0 and float(rows[0]["bubble_sim_float"]) < 0.2
