"""Layer -> virtual-stage partitioner (SURVEY §7 step 3, §8(b) partitioner
row): uniform rule, explicit counts, and the cost-balanced variant."""
from fractions import Fraction

import pytest

from paper_2410_19367_b200 import schedule as ps
from paper_2410_19367_b200.model import CONFIGS, balanced_counts, device_loads, stage_costs, stage_partition
from paper_2410_19367_b200.schedule import list_schedule


def _makespan(cfg, sched, counts):
    cost = [Fraction(round(x / 1e6)) for x in stage_costs(cfg, counts)]
    dur = lambda t: cost[t.stage] * (1 if t.kind.value == "F" else 2)  # noqa: E731
    starts = list_schedule(sched.per_device, sched.dependencies, dur)
    return max(st + dur(t) for t, st in starts.items())


def test_explicit_counts_and_validation():
    cfg = CONFIGS["tiny"]
    plans = stage_partition(cfg, 8, [2, 0, 1, 1, 1, 1, 2, 0])
    assert [p.halfblocks for p in plans] == [(0, 1), (), (2,), (3,), (4,), (5,), (6, 7), ()]
    assert plans[0].embed and plans[-1].head and not plans[3].embed
    with pytest.raises(ValueError):
        stage_partition(cfg, 8, [1] * 7)
    with pytest.raises(ValueError):
        stage_partition(cfg, 8, [2, 2, 2, 2, 0, 0, 0, -1])


@pytest.mark.parametrize("name,D,N", [("gpt-1.3b", 8, 16), ("bert-large", 4, 8), ("gpt-1.3b", 4, 8)])
def test_balanced_partition_shortens_modelled_pipeline(name, D, N):
    """The cost-balanced split never lengthens the modelled replay and, at
    GPT/BERT sizes where the LM head weighs 2-4 half-blocks, shortens it."""
    cfg = CONFIGS[name]
    for sched in (ps.build_bitpipe(D, N), ps.build_bitpipe(D, N, policy=ps.paper_policy(D))):
        uni = [len(p.halfblocks) for p in stage_partition(cfg, sched.num_stages)]
        bal = balanced_counts(cfg, sched)
        assert sum(bal) == 2 * cfg.layers and min(bal) >= 0
        assert bal == balanced_counts(cfg, sched)  # deterministic
        assert _makespan(cfg, sched, bal) < _makespan(cfg, sched, uni)
        maps = [sched.stage_map(d) for d in sched.directions]
        assert max(device_loads(cfg, bal, maps)) <= max(device_loads(cfg, uni, maps))


def test_device_loads_v_map_symmetry():
    """Both directions place the same partition mirrored: device d and
    D-1-d carry the same stages (V map, schedules.py:96-108)."""
    cfg = CONFIGS["gpt-1.3b"]
    sched = ps.build_bitpipe(8, 16)
    maps = [sched.stage_map(d) for d in sched.directions]
    ld = device_loads(cfg, [3] * 16, maps)
    assert all(abs(ld[d] - ld[7 - d]) < 1e-6 * ld[d] for d in range(8))
    assert ld[0] > ld[1]  # embedding + LM head stages sit on devices 0 and 7


def test_policy_search_generalises_f2():
    """Generalised F2: the policy search over the
    reference engine's layout policies finds the analytic-bubble order at
    D=8 N=16 (the F2 gate 10) and near-analytic orders where no gate is known
    (D=6); with the PAPER Table 2 activation bound D M_a it still beats the
    default order."""
    pol, s, b, peak = ps.search_bitpipe_policy(8, 16)
    assert b == ps.analytic_bubble_ratio(ps.ApproachId.BITPIPE, 8, 16) and pol.gate_stage == 10 and not pol.defer
    assert peak == 12  # 12 M_a at N=16
    assert ps.dump_schedule(s) == ps.dump_schedule(ps.build_bitpipe(8, 16, policy=ps.paper_policy(8)))
    _, s6, b6, _ = ps.search_bitpipe_policy(6, 12)
    assert b6 < ps.canonical_bubble(ps.build_bitpipe(6, 12)) and b6 < Fraction(12, 100)
    _, sc, bc, pc = ps.search_bitpipe_policy(8, 16, max_peak=8)
    assert pc <= 8 and max(ps.peak_activations(sc)) <= 8
    assert bc < ps.canonical_bubble(ps.build_bitpipe(8, 16))
    with pytest.raises(ValueError):
        ps.search_bitpipe_policy(4, 8, max_peak=1)


def test_peak_activations_default_order():
    """Non-EF BitPipe peaks lie in PAPER Table 2's [(D+3)/2, D] M_a (D=4 N=8 gives 3.5, 4, 4, 3.5)."""
    assert ps.peak_activations(ps.build_bitpipe(4, 8)) == [Fraction(7, 2), 4, 4, Fraction(7, 2)]
