"""bench.py --impl reference (CPU oracle arm) prints the contract JSON line."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "small",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "small",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_gpus_flag_self_launches_ranks():
    """``--gpus 2`` without a torchrun environment launches 2 ranks itself
    (the reference arm runs on CPU, so this needs no GPU): exactly one JSON
    line, from rank 0, on the configuration of a 2-GPU run (D = 2)."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "small",
                          "--gpus", "2", "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and "D=2" in line["config"]["workload"]


@pytest.mark.gpu
def test_multirank_bench_on_one_gpu():
    """``--gpus 4`` through the self-launcher with every rank on cuda:0
    (BP_SHARE_GPU=1): the distributed Trainer over the peer transport, the
    max-over-ranks device timing and the measured multi-rank bubble all run
    and rank 0 prints one contract line."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    env.update(BP_SHARE_GPU="1", BP_SKIP_CPU_BASELINE="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "small", "--gpus", "4",
                          "--N", "8", "--steps", "2", "--warmup", "3"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 4 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["transport"].startswith("peer") and "SHARE ONE GPU" in line["transport"]
    m = line["bubble"]["measured"]
    assert 0.0 <= m["bubble"] < 1.0 and len(m["busy_ms_per_rank"]) == 4


@pytest.mark.gpu
def test_single_gpu_bench_line():
    """``bench.py`` (our arm, N = 1) on a small configuration: the contract
    keys, the roofline / cpu_baseline / e2e / clocks objects and a positive
    native launch count."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "small", "--D", "4", "--N", "8",
                          "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "cpu_baseline", "gpu_launches", "clocks"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3 and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert line["roofline"]["unit"] == "TFLOP/s" and 0 < line["roofline"]["frac"] < 1.2
    assert line["cpu_baseline"]["cores"] >= 1 and line["gpu_launches"] > 0
    assert "workload" in line["config"]
