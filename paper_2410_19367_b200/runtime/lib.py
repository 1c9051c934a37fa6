"""ctypes binding of ``libbitpipe_b200.so`` (declared in ``include/bitpipe.h``).

This is the only way the host driver reaches the GPU kernels.  There is no
fallback: if the library is missing or a call fails, a RuntimeError is
raised with the library's own error text.
"""
from __future__ import annotations

import ctypes
import os
import threading

__all__ = ["lib", "GemmArgs", "check", "LIB_PATH", "BP_F32", "BP_BF16", "EPI_NONE", "EPI_GELU", "EPI_DGELU",
           "OPT_ATTN_EXACT", "OPT_GEMM_SIMT", "OPT_GEMM_MODE",
           "OPT_STREAM_K", "OPT_GEMM_WIDE", "OPT_GEMM_DEBUG", "OPT_GEMM_TMA_STORE", "OPT_LN_UNFUSED",
           "OPT_LN_BWD_MODE", "OPT_ATTN_FWD_MODE", "OPT_GEMM_OCC", "OPT_GEMM_GRID", "OPT_GEMM_BN", "OPT_ATTN_BWD_MODE",
           "OPT_GEMM_EPI_WARPS", "OPT_ATTN_FWD_EXF", "OPT_GEMM_L2_HINTS", "OPT_LN_CTAS_PER_SM",
           "OPT_GEMM_PICK"]

LIB_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "libbitpipe_b200.so")

BP_F32, BP_BF16 = 0, 1
EPI_NONE, EPI_GELU, EPI_DGELU = 0, 1, 2
OPT_ATTN_EXACT, OPT_GEMM_SIMT, OPT_GEMM_MODE, OPT_STREAM_K, OPT_GEMM_WIDE = 1, 2, 3, 4, 5
OPT_GEMM_DEBUG, OPT_GEMM_TMA_STORE, OPT_LN_UNFUSED, OPT_LN_BWD_MODE, OPT_ATTN_FWD_MODE = 6, 7, 8, 10, 11
OPT_GEMM_OCC, OPT_GEMM_GRID, OPT_GEMM_BN, OPT_ATTN_BWD_MODE, OPT_GEMM_EPI_WARPS = 12, 13, 14, 15, 16
OPT_ATTN_FWD_EXF, OPT_GEMM_L2_HINTS, OPT_LN_CTAS_PER_SM, OPT_GEMM_PICK = 17, 18, 9, 19
ABI_VERSION = 2

_vp = ctypes.c_void_p
_i32, _i64, _f32 = ctypes.c_int, ctypes.c_int64, ctypes.c_float


class GemmArgs(ctypes.Structure):
    _fields_ = [
        ("M", _i32), ("N", _i32), ("K", _i32), ("in_dtype", _i32),
        ("a_kmajor", _i32), ("b_kmajor", _i32),
        ("A", _vp), ("lda", _i64), ("B", _vp), ("ldb", _i64),
        ("C", _vp), ("ldc", _i64), ("c_dtype", _i32),
        ("alpha", _f32), ("beta", _f32),
        ("bias", _vp), ("residual", _vp), ("ldr", _i64),
        ("aux", _vp), ("ldaux", _i64),
        ("epilogue", _i32), ("force_simt", _i32), ("colsum", _vp),
    ]


_SIGS = {
    "bp_abi_version": (_i32, []),
    "bp_last_error": (ctypes.c_char_p, []),
    "bp_sm_count": (_i32, [_i32]),
    "bp_tc_available": (_i32, []),
    "bp_launch_count": (ctypes.c_ulonglong, []),
    "bp_set_option": (_i32, [_i32, _i32]),
    "bp_gemm": (_i32, [ctypes.POINTER(GemmArgs), _vp]),
    "bp_layernorm_fwd": (_i32, [_i32, _i32, _i32, _vp, _vp, _vp, _f32, _vp, _vp, _vp, _vp]),
    "bp_layernorm_bwd": (_i32, [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bp_layernorm_bwd_ex": (_i32, [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bp_colsum_acc": (_i32, [_i32, _i32, _i32, _vp, _i64, _vp, _vp]),
    "bp_embed_fwd": (_i32, [_i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "bp_embed_bwd": (_i32, [_i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "bp_xent_fwd_bwd": (_i32, [_i32, _i32, _i32, _vp, _i64, _vp, _f32, _f32, _vp, _vp]),
    "bp_cast": (_i32, [_i32, _i32, _i64, _vp, _vp, _vp]),
    "bp_attn_workspace_bytes": (_i64, [_i32, _i32, _i32, _i32]),
    "bp_attn_fwd": (_i32, [_i32, _i32, _i32, _i32, _i32, _i32, _f32, _vp, _vp, _vp, _vp]),
    "bp_attn_bwd": (_i32, [_i32, _i32, _i32, _i32, _i32, _i32, _f32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bp_attn_bwd_ex": (_i32, [_i32, _i32, _i32, _i32, _i32, _i32, _f32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bp_adam": (_i32, [_i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _f32, _f32, _f32, _f32, _f32, _i32, _f32,
                       _vp]),
    "bp_adam_dev": (_i32, [_i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _f32, _f32, _f32, _f32, _f32, _i32, _vp,
                           _f32, _vp]),
    # include/bitpipe_comm.h: runtime context (NCCL via dlopen), slots, events, graphs
    "bp_comm_available": (_i32, []),
    "bp_nccl_unique_id": (_i32, [_vp]),
    "bp_init": (_i32, [_i32, _i32, _vp, _i32, ctypes.POINTER(_vp)]),
    "bp_comm_split": (_i32, [_vp, _i32, _i32, ctypes.POINTER(_vp)]),
    "bp_comm_rank": (_i32, [_vp]),
    "bp_comm_size": (_i32, [_vp]),
    "bp_slots_alloc": (_i32, [_vp, ctypes.c_size_t, _i32, ctypes.POINTER(_vp)]),
    "bp_slot_stride": (ctypes.c_size_t, [ctypes.c_size_t]),
    "bp_send": (_i32, [_vp, _i32, _vp, ctypes.c_size_t, _vp]),
    "bp_recv": (_i32, [_vp, _i32, _vp, ctypes.c_size_t, _vp]),
    "bp_group_start": (_i32, []),
    "bp_group_end": (_i32, []),
    "bp_allreduce_mean": (_i32, [_vp, _vp, ctypes.c_size_t, _i32, _vp]),
    "bp_destroy": (_i32, [_vp]),
    "bp_event_create": (_i32, [ctypes.POINTER(_vp)]),
    "bp_event_record": (_i32, [_vp, _vp]),
    "bp_stream_wait_event": (_i32, [_vp, _vp]),
    "bp_event_destroy": (_i32, [_vp]),
    "bp_graph_begin": (_i32, [_vp]),
    "bp_graph_end": (_i32, [_vp, ctypes.POINTER(_vp)]),
    "bp_graph_launch": (_i32, [_vp, _vp]),
    "bp_graph_destroy": (_i32, [_vp]),
    # include/bitpipe_comm.h, peer memory: CUDA IPC, peer copies, stream-ordered flags
    "bp_ipc_export": (_i32, [_vp, _vp, ctypes.POINTER(ctypes.c_size_t)]),
    "bp_ipc_open": (_i32, [_vp, ctypes.POINTER(_vp)]),
    "bp_ipc_close": (_i32, [_vp]),
    "bp_memcpy_async": (_i32, [_vp, _vp, ctypes.c_size_t, _vp]),
    "bp_flag_set": (_i32, [_vp, _vp, ctypes.c_uint32]),
    "bp_flag_wait": (_i32, [_vp, _vp, ctypes.c_uint32]),
    "bp_flag_wait_spin": (_i32, [_vp, _vp, ctypes.c_uint32]),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def lib() -> ctypes.CDLL:
    """Load (once) and return the library; RuntimeError if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"BitPipe CUDA library not built: {LIB_PATH} missing "
                                   f"(run `make` or __graft_entry__.build())")
            h = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            if h.bp_abi_version() != ABI_VERSION:
                raise RuntimeError("libbitpipe_b200.so ABI version mismatch")
            # A/B switches for measurements (tools/, bench): BP_GEMM_OCC=0/1/2
            for env, opt in (("BP_GEMM_OCC", OPT_GEMM_OCC), ("BP_GEMM_GRID", OPT_GEMM_GRID),
                             ("BP_GEMM_BN", OPT_GEMM_BN),
                             ("BP_ATTN_BWD_MODE", OPT_ATTN_BWD_MODE), ("BP_GEMM_EW", OPT_GEMM_EPI_WARPS),
                             ("BP_ATTN_FWD_EXF", OPT_ATTN_FWD_EXF),
                             ("BP_GEMM_PICK", OPT_GEMM_PICK)):
                if os.environ.get(env, "") != "":
                    h.bp_set_option(opt, int(os.environ[env]))
            _lib = h
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().bp_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed (code {rc}): {msg}")
