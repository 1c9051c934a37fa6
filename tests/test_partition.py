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


# -- communication accounting (PAPER Appendix C Table 6)
def test_comm_accounting_counts():
    from paper_2410_19367_b200 import schedule as ps
    prof = lambda N: ps.ModelProfile(1, N, 2048, 2048)  # noqa: E731
    for D in (2, 4, 8):
        for N in (D, 2 * D, 4 * D):
            b = ps.comm_accounting(ps.build_bitpipe(D, N), prof(N), grad_bytes_per_stage=3)
            assert b.p2p_messages == N * (4 * D - 4)
            assert b.local_copies == 2 * N                       # the V fold, F and B, every micro-batch
            assert b.p2p_bytes == b.p2p_messages * 2 * 2048 * 2048
            assert b.allreduce_groups == (D // 2) * 4            # 2v stages per replica pair
            assert b.allreduce_bytes == 4 * 3
            assert set(b.per_link) == {(d, d + 1) for d in range(D - 1)} | {(d + 1, d) for d in range(D - 1)}
            il = ps.comm_accounting(ps.build_interleaved_looping(D, N), prof(N))
            # looping count minus the local-copy edges
            assert il.p2p_messages - b.p2p_messages == 2 * N and il.local_copies == 0
            assert ps.comm_accounting(ps.build_1f1b(D, N), prof(N)).p2p_messages == N * 2 * (D - 1)
    assert ps.comm_accounting(ps.build_1f1b(1, 4), prof(4)).p2p_messages == 0   # D=1: all local
    # intra / inter split by devices_per_node: D=8 over two 4-GPU nodes, only the 3<->4 link crosses
    c = ps.comm_accounting(ps.build_bitpipe(8, 16), prof(16), ps.ClusterSpec(8, devices_per_node=4))
    assert c.p2p_bytes_inter == (c.per_link[(3, 4)] + c.per_link[(4, 3)]) * 2 * 2048 * 2048
    assert c.p2p_bytes_intra + c.p2p_bytes_inter == c.p2p_bytes


def test_analytic_comm_time_table6():
    from fractions import Fraction
    import pytest
    from paper_2410_19367_b200 import schedule as ps
    A = ps.ApproachId
    cl = ps.ClusterSpec(4, intra_node_bandwidth=200e9, inter_node_bandwidth=25e9)
    prof = ps.ModelProfile(1, 4, 1024, 3072)   # message_size = 6,291,456 B
    assert ps.message_size(prof) == 6291456
    # DAPPLE D=4 N=4 -> 14 messages, ~3.52 ms
    assert ps.analytic_comm_count(A.DAPPLE_1F1B, 4, 4) == 14
    assert abs(ps.analytic_comm_time(A.DAPPLE_1F1B, 4, 4, prof, cl) - 14 * 6291456 / 25e9) < 1e-15
    assert ps.analytic_comm_count(A.INTERLEAVED_LOOPING, 4, 4) == 28
    # BitPipe's P2P term is exactly 2x Chimera's; allreduce terms equal
    for D, N in ((4, 4), (8, 16), (8, 32)):
        mg = 1.5e9
        b = ps.analytic_comm_time(A.BITPIPE, D, N, prof, cl, mg) - mg / 200e9
        c = ps.analytic_comm_time(A.CHIMERA, D, N, prof, cl, mg) - mg / 200e9
        assert abs(b - 2 * c) < 1e-12
        assert Fraction(ps.analytic_comm_count(A.BITPIPE, D, N), ps.analytic_comm_count(A.DAPPLE_1F1B, D, N)) == 2
    with pytest.raises(ps.errors.UnsupportedCombination):
        ps.analytic_comm_time(A.GPIPE, 4, 4, prof, cl)


def _synthetic_costs():
    return {"F": {"attn": 0.16, "mlp": 0.17, "head": 0.45, "embed": 0.03},
            "B": {"attn": 0.27, "mlp": 0.31, "head": 0.67, "embed": 0.03},
            "Bd": {"attn": 0.20, "mlp": 0.16, "head": 0.27, "embed": 0.02},
            "W": {"attn": 0.05, "mlp": 0.10, "head": 0.33, "embed": 0.01}}


def test_fit_task_costs_recovers_a_linear_table():
    """The least-squares fit of measured task times (model.fit_task_costs)
    returns the per-term table that generated them (W per micro-batch)."""
    from paper_2410_19367_b200.model import fit_task_costs, modelled_task_times
    sched = ps.build_bitpipe(8, 16, policy=ps.paper_policy(8))
    counts = [3, 3, 3, 2, 4, 3, 3, 3, 3, 3, 3, 2, 4, 4, 4, 1]
    costs = _synthetic_costs()
    fit = fit_task_costs(counts, modelled_task_times(counts, costs, sched), 8)
    for kind in costs:
        for term in costs[kind]:
            assert fit[kind][term] == pytest.approx(costs[kind][term], abs=1e-9)


@pytest.mark.parametrize("name,D,N", [("gpt-1.3b", 8, 16), ("bert-large", 4, 8)])
def test_calibrated_partition_shortens_the_as_executed_replay(name, D, N):
    """The measured-cost partition (model.calibrated_counts) never lengthens
    the as-executed replay of its start, keeps every non-head stage
    non-empty, and is deterministic."""
    from paper_2410_19367_b200.model import calibrated_counts, modelled_task_times, resolve_partition
    from paper_2410_19367_b200.schedule.analysis import replay_times
    cfg = CONFIGS[name]
    sched = ps.build_bitpipe(D, N, policy=ps.paper_policy(D))
    costs = _synthetic_costs()
    start = resolve_partition(cfg, sched, "balanced")
    c = calibrated_counts(cfg, sched, costs, start=start)
    assert sum(c) == 2 * cfg.layers and min(c[:-1]) >= 1 and c[-1] >= 0
    assert c == calibrated_counts(cfg, sched, costs, start=start)
    mk = lambda cc: replay_times(sched, modelled_task_times(cc, costs, sched), True)["makespan_ms"]  # noqa: E731
    assert mk(c) <= mk(start)


def test_resolve_partition_kinds():
    from paper_2410_19367_b200.model import load_calibration, resolve_partition
    cfg = CONFIGS["tiny"]
    sched = ps.build_bitpipe(4, 8)
    assert resolve_partition(cfg, sched, "uniform") == [len(p.halfblocks) for p in stage_partition(cfg, 8)]
    assert resolve_partition(cfg, sched, [2, 0, 1, 1, 1, 1, 2, 0]) == [2, 0, 1, 1, 1, 1, 2, 0]
    assert load_calibration("tiny") is None
    assert resolve_partition(cfg, sched, "auto") == resolve_partition(cfg, sched, "balanced")
    with pytest.raises(ValueError, match="calibration"):
        resolve_partition(cfg, sched, "calibrated")
    # the committed B200 tables load and give valid partitions
    for name, D, N in (("gpt-1.3b", 8, 16), ("bert-large", 4, 8)):
        assert load_calibration(name) is not None
        c = resolve_partition(CONFIGS[name], ps.build_bitpipe(D, N, policy=ps.paper_policy(D)), "auto")
        assert sum(c) == 2 * CONFIGS[name].layers
