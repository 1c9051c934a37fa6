"""Host-side executor logic that needs no GPU."""
import pytest
import torch

from paper_2410_19367_b200.runtime.executor import choose_deferred_stages


def test_all_stages_deferred_when_slots_fit():
    assert choose_deferred_stages({0: 10, 1: 20, 2: 30}, {0: 1, 1: 1, 2: 1}, 60) == {0, 1, 2}


def test_greedy_by_work_per_byte_under_budget():
    sizes = {0: 40, 1: 40, 2: 10, 3: 0}
    work = {0: 80, 1: 40, 2: 30, 3: 5}
    # work / byte: stage 2 (3.0), stage 0 (2.0), stage 1 (1.0); empty slot sets are never "deferred"
    assert choose_deferred_stages(sizes, work, 55) == {2, 0}
    assert choose_deferred_stages(sizes, work, 5) == set()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the CPU-only failure mode")
def test_train_step_fails_loudly_without_a_gpu():
    """No CPU fallback: the SPEC entry refuses to run without CUDA."""
    from paper_2410_19367_b200 import build_bitpipe
    from paper_2410_19367_b200.model import CONFIGS, synthetic_batch
    from paper_2410_19367_b200.runtime.api import train_step
    with pytest.raises(RuntimeError, match="CUDA"):
        train_step(build_bitpipe(2, 4), "tiny", synthetic_batch(CONFIGS["tiny"], 4))


def _unit_times(sched, F=1.0, B=2.0, Bd=None, W=0.0):
    out = {}
    for dr in sched.directions:
        for s in range(sched.num_stages):
            out[(dr, s, "F")], out[(dr, s, "B")] = F, B
            out[(dr, s, "Bd")] = B if Bd is None else Bd
            out[(dr, s, "W")] = W
    return out


@pytest.mark.parametrize("D,N", [(4, 8), (8, 16)])
def test_replay_unit_times_is_the_canonical_bubble(D, N):
    """F = 1, B = 2 replays the paper order at its analytic bubble (PAPER Table 2:
    (D-2)/(3N/2+D-2) for BitPipe, = 1/9 at D=8 N=16)."""
    from fractions import Fraction

    from paper_2410_19367_b200 import schedule as ps
    from paper_2410_19367_b200.schedule.analysis import replay_times
    sched = ps.build_bitpipe(D, N, policy=ps.paper_policy(D))
    r = replay_times(sched, _unit_times(sched))
    assert abs(r["bubble"] - float(ps.canonical_bubble(sched))) < 1e-12
    # deferred form with no weight-gradient work and unchanged B: identical replay
    r2 = replay_times(sched, _unit_times(sched, W=0.0), deferred_w=True)
    assert r2 == r


def test_replay_deferred_weight_gradients_fill_the_drain():
    """B = 1 (input-gradient chain) + W = 1 per micro-batch, deferred into one
    block per stage replica after its last backward: the same busy time as
    B = 2, a shorter makespan (the drain is filled), a smaller bubble."""
    from paper_2410_19367_b200 import schedule as ps
    from paper_2410_19367_b200.schedule.analysis import replay_times
    D, N = 8, 16
    sched = ps.build_bitpipe(D, N, policy=ps.paper_policy(D))
    per_mb = _unit_times(sched)
    n_rep = N // 2
    dfr = _unit_times(sched, Bd=1.0, W=1.0 * n_rep)
    a = replay_times(sched, per_mb)
    b = replay_times(sched, dfr, deferred_w=True)
    assert sum(a["busy_ms_per_device"]) == pytest.approx(sum(b["busy_ms_per_device"]))
    assert b["makespan_ms"] < a["makespan_ms"]
    assert b["bubble"] < a["bubble"]
