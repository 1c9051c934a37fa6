"""GEMM epilogue probe on the 1.3B shapes: per-thread stores (TMA_STORE=0)
vs the TMA-store epilogue (1) vs TMEM drained with no stores (debug)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import ops
from paper_2410_19367_b200.runtime.ops import EPI_GELU
from paper_2410_19367_b200.runtime.lib import OPT_GEMM_DEBUG, OPT_GEMM_TMA_STORE


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


h = 2048
for name, M, N, K, ak, bk, kind in [("qkv fprop", 2048, 3 * h, h, True, True, "bias"),
                                    ("proj fprop", 2048, h, h, True, True, "res"),
                                    ("fc1 fprop", 2048, 4 * h, h, True, True, "gelu"),
                                    ("fc2 fprop", 2048, h, 4 * h, True, True, "res"),
                                    ("fc1 dgrad", 2048, h, 4 * h, True, False, "plain"),
                                    ("fc2 dgrad", 2048, 4 * h, h, True, False, "dgelu"),
                                    ("fc1 wgrad", 4 * h, h, 2048, False, False, "acc"),
                                    ("head fprop", 2048, 50304, h, True, True, "plain"),
                                    ("head wgrad", 50304, h, 2048, False, False, "acc"),
                                    ("sq 8192", 8192, 8192, 8192, True, True, "plain")]:
    A = (torch.randn(M, K) if ak else torch.randn(K, M)).cuda().bfloat16()
    B = (torch.randn(N, K) if bk else torch.randn(K, N)).cuda().bfloat16()
    acc = kind == "acc"
    C = torch.zeros(M, N, device="cuda", dtype=torch.float32 if acc else torch.bfloat16)
    bias = torch.randn(N, device="cuda").bfloat16() if kind in ("bias", "res", "gelu") else None
    res = torch.randn(M, N, device="cuda").bfloat16() if kind == "res" else None
    aux = torch.randn(M, N, device="cuda").bfloat16() if kind in ("gelu", "dgelu") else None
    epi = {"gelu": EPI_GELU, "dgelu": 2}.get(kind, 0)
    out = []
    for tma, dbg in ((0, 0), (1, 0), (1, 1)):
        ops.set_option(OPT_GEMM_TMA_STORE, tma)
        ops.set_option(OPT_GEMM_DEBUG, dbg)
        ms = timeit(lambda: ops.gemm(A, B, C, a_kmajor=ak, b_kmajor=bk, beta=1.0 if acc else 0.0, bias=bias,
                                     residual=res, aux=aux, epilogue=epi))
        out.append((ms * 1e3, 2 * M * N * K / ms / 1e9))
    ops.set_option(OPT_GEMM_TMA_STORE, 1)
    ops.set_option(OPT_GEMM_DEBUG, 0)
    print(f"{name:10s} {kind:5s} thread-store {out[0][0]:7.1f} us {out[0][1]:6.0f} TF/s | tma-store "
          f"{out[1][0]:7.1f} us {out[1][1]:6.0f} TF/s | no-store {out[2][0]:7.1f} us {out[2][1]:6.0f} TF/s",
          flush=True)
