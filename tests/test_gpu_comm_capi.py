"""The runtime-context C ABI (include/bitpipe_comm.h) on one GPU: a 1-rank
NCCL communicator and a split of it, the replica-mean all-reduce (identity
over one rank), a self send / receive pair in one NCCL group into a message
slot, events, and a CUDA graph of library kernels captured and replayed
through bp_graph_*."""
import ctypes as C

import pytest
import torch

from paper_2410_19367_b200.runtime import lib as L
from paper_2410_19367_b200.runtime import ops

pytestmark = pytest.mark.gpu


def _ok(rc, what):
    assert rc == 0, (what, L.lib().bp_last_error())


@pytest.fixture()
def ctx():
    h = L.lib()
    if not h.bp_comm_available():
        pytest.skip("no NCCL library")
    uid = (C.c_ubyte * 128)()
    _ok(h.bp_nccl_unique_id(uid), "unique id")
    c = C.c_void_p()
    _ok(h.bp_init(0, 1, uid, torch.cuda.current_device(), C.byref(c)), "bp_init")
    assert h.bp_comm_rank(c) == 0 and h.bp_comm_size(c) == 1
    yield c
    _ok(h.bp_destroy(c), "bp_destroy")


def test_allreduce_mean_split_and_self_p2p(ctx):
    h = L.lib()
    st = torch.cuda.Stream()
    s = C.c_void_p(st.cuda_stream)
    sub = C.c_void_p()
    _ok(h.bp_comm_split(ctx, 0, 0, C.byref(sub)), "split")
    assert sub.value and h.bp_comm_size(sub) == 1 and h.bp_comm_rank(sub) == 0
    for dt, tdt in ((L.BP_F32, torch.float32), (L.BP_BF16, torch.bfloat16)):
        x = torch.randn(100003, device="cuda").to(tdt)
        ref = x.clone()
        torch.cuda.synchronize()
        _ok(h.bp_allreduce_mean(sub, C.c_void_p(x.data_ptr()), x.numel(), dt, s), "allreduce")
        st.synchronize()
        assert torch.equal(x, ref)  # mean over one rank
    # message slots + a self send / receive in one group
    nbytes = 3 * 2048 * 2
    base = C.c_void_p()
    _ok(h.bp_slots_alloc(ctx, nbytes, 4, C.byref(base)), "slots")
    stride = h.bp_slot_stride(nbytes)
    msg = torch.randn(3, 2048, device="cuda").bfloat16()
    torch.cuda.synchronize()
    slot2 = C.c_void_p(base.value + 2 * stride)
    _ok(h.bp_group_start(), "group start")
    _ok(h.bp_send(ctx, 0, C.c_void_p(msg.data_ptr()), nbytes, s), "send")
    _ok(h.bp_recv(ctx, 0, slot2, nbytes, s), "recv")
    _ok(h.bp_group_end(), "group end")
    got = torch.empty_like(msg)
    ev = C.c_void_p()
    _ok(h.bp_event_create(C.byref(ev)), "event")
    _ok(h.bp_event_record(ev, s), "record")
    main = torch.cuda.current_stream()
    _ok(h.bp_stream_wait_event(C.c_void_p(main.cuda_stream), ev), "wait")
    # and back out of the slot into a tensor, ordered behind the event
    _ok(h.bp_group_start(), "group start")
    _ok(h.bp_send(ctx, 0, slot2, nbytes, C.c_void_p(main.cuda_stream)), "send")
    _ok(h.bp_recv(ctx, 0, C.c_void_p(got.data_ptr()), nbytes, C.c_void_p(main.cuda_stream)), "recv")
    _ok(h.bp_group_end(), "group end")
    torch.cuda.synchronize()
    assert torch.equal(got, msg)
    _ok(h.bp_event_destroy(ev), "event destroy")
    _ok(h.bp_destroy(sub), "destroy sub")


def test_graph_capture_and_replay_of_library_kernels():
    h = L.lib()
    st = torch.cuda.Stream()
    s = C.c_void_p(st.cuda_stream)
    x = torch.randn(4096, 512, device="cuda")
    y = torch.empty(4096, 512, device="cuda", dtype=torch.bfloat16)
    z = torch.empty(4096, 512, device="cuda")
    torch.cuda.synchronize()
    _ok(h.bp_graph_begin(s), "graph begin")
    ops.cast(x, y, stream=st)
    ops.cast(y, z, stream=st)
    ge = C.c_void_p()
    _ok(h.bp_graph_end(s, C.byref(ge)), "graph end")
    for scale in (1.0, -3.0):
        x.mul_(scale)
        torch.cuda.synchronize()
        _ok(h.bp_graph_launch(ge, s), "graph launch")
        st.synchronize()
        assert torch.equal(z, x.bfloat16().float())
    _ok(h.bp_graph_destroy(ge), "graph destroy")
