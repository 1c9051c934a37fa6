"""The C-ABI library loads on a CPU-only host and exports exactly what
include/bitpipe.h and include/bitpipe_comm.h declare (no compute calls
without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in ("bitpipe.h", "bitpipe_comm.h")]


def declared():
    text = "".join(open(h).read() for h in HEADERS)
    return sorted(set(re.findall(r"BP_API\s+[\w\s\*]+?\b(bp_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared()
    assert "bp_gemm" in names and "bp_attn_bwd" in names and "bp_adam" in names
    assert len(names) >= 18


def test_library_exports_every_declared_symbol():
    from paper_2410_19367_b200.runtime import lib as L
    if not os.path.exists(L.LIB_PATH):
        pytest.skip("library not built (run make)")
    h = ctypes.CDLL(L.LIB_PATH)
    for n in declared():
        assert hasattr(h, n), n
    # the Python binding covers the same surface
    assert set(declared()) == set(L.EXPORTED)
    h.bp_abi_version.restype = ctypes.c_int
    assert h.bp_abi_version() == L.ABI_VERSION


def test_error_path_without_gpu():
    """Bad arguments are rejected with an error code and message, never ignored."""
    from paper_2410_19367_b200.runtime import lib as L
    if not os.path.exists(L.LIB_PATH):
        pytest.skip("library not built")
    h = L.lib()
    g = L.GemmArgs()
    g.M, g.N, g.K = 0, 16, 16
    rc = h.bp_gemm(ctypes.byref(g), None)
    assert rc == 1 and b"bad shape" in h.bp_last_error()


def test_comm_context_without_gpu():
    """The runtime context resolves NCCL at run time (no link dependency);
    argument errors come back as codes + messages; a unique id needs no GPU."""
    import ctypes as C

    import torch  # noqa: F401  -- torch's NCCL first (see bitpipe_comm.h)
    from paper_2410_19367_b200.runtime import lib as L
    if not os.path.exists(L.LIB_PATH):
        pytest.skip("library not built")
    h = L.lib()
    assert "bp_allreduce_mean" in declared() and "bp_graph_launch" in declared()
    assert h.bp_slot_stride(1) == 256 and h.bp_slot_stride(256) == 256 and h.bp_slot_stride(8 << 20) == 8 << 20
    out = C.c_void_p()
    assert h.bp_slots_alloc(None, 16, 1, C.byref(out)) == 1 and b"invalid" in h.bp_last_error()
    if not h.bp_comm_available():
        pytest.skip("no NCCL library on this host")
    assert h.bp_init(0, 1, None, 0, C.byref(out)) == 1
    uid = (C.c_ubyte * 128)()
    assert h.bp_nccl_unique_id(uid) == 0
    assert any(uid)
