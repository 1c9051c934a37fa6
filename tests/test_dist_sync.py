"""Eager replica-pair sync ordering: the two holders of a
stage reach their last backwards of their shared stages in different
orders, so collectives chained on one stream per rank deadlock; the
executor gives every stage its own optimizer stream."""
import pytest

from paper_2410_19367_b200 import schedule as ps
from paper_2410_19367_b200.runtime.distributed import DistContext, stage_sync_orders, sync_order_acyclic


@pytest.mark.parametrize("D,N", [(4, 8), (8, 16)])
def test_default_bitpipe_orders_would_deadlock_on_one_stream(D, N):
    sched = ps.build_bitpipe(D, N)
    orders = stage_sync_orders(sched)
    assert orders[0] != orders[D - 1]          # e.g. D=4 N=8: [7, 0, 4, 3] vs [4, 3, 7, 0]
    assert not sync_order_acyclic(sched, shared_stream=True)
    assert sync_order_acyclic(sched, shared_stream=False)


def _schedules():
    for D in (2, 4, 8):
        for N in (D, 2 * D, 4 * D):
            yield ps.build_bitpipe(D, N)
            if N >= 2 * D:
                yield ps.build_bitpipe(D, N, early_forward=True)
            if D in ps.PAPER_GATE_STAGE:
                yield ps.build_bitpipe(D, N, policy=ps.paper_policy(D))
            yield ps.build(ps.ApproachId.CHIMERA, D, N)
            yield ps.build(ps.ApproachId.DAPPLE_1F1B, D, N)


def test_every_stage_sync_goes_to_its_own_stream():
    """DistContext.sync_stage issues stage s's all-reduce + AdamW on
    trainer.stage_stream(s), never on a stream shared with another stage."""
    calls = []

    class Ev:
        pass

    class Stream:
        def __init__(self, s):
            self.s = s

        def wait_event(self, ev):
            pass

    class FakeTrainer:
        stage_params = {}

        def stage_stream(self, s):
            return Stream(s)

        def _adam(self, key, grads, outs, st, grad_scale=1.0):
            calls.append((key[1], st.s))

    class SP:
        grad = flat = None

    ctx = DistContext(0, 2, cuda=False)
    ctx.allreduce_stage = lambda s, t, stream=None: (calls.append(("ar", s, stream.s)), 2)[1]
    tr = FakeTrainer()
    for s in (3, 0, 2):
        tr.stage_params[("down", s)] = SP()
        ctx.sync_stage(tr, "down", s, Ev())
    assert [c for c in calls if c[0] != "ar"] == [(3, 3), (0, 0), (2, 2)]
    assert [c for c in calls if c[0] == "ar"] == [("ar", 3, 3), ("ar", 0, 0), ("ar", 2, 2)]


def test_sync_orders_cover_every_builder():
    for sched in _schedules():
        orders = stage_sync_orders(sched)
        held = {d: sorted({(t.direction, t.stage) for t in row if t.kind is ps.TaskKind.BACKWARD})
                for d, row in enumerate(sched.per_device)}
        for d in range(sched.D):
            assert sorted(orders[d]) == sorted(s for _dr, s in held[d])
