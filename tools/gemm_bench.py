"""Micro-benchmark of the tcgen05 GEMM against cuBLAS (torch.matmul) on the
GPT-1.3B per-micro-batch shapes.  Prints one line per shape."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import ops

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

T, h, f, V = 2048, 2048, 8192, 50304
cases = [  # name, M, N, K, a_kmajor, b_kmajor, fp32-accumulate
    ("qkv fprop", T, 3 * h, h, True, True, False),
    ("proj fprop", T, h, h, True, True, False),
    ("fc1 fprop", T, f, h, True, True, False),
    ("fc2 fprop", T, h, f, True, True, False),
    ("lm fprop", T, V, h, True, True, False),
    ("fc1 dgrad", T, h, f, True, False, False),
    ("fc2 dgrad", T, f, h, True, False, False),
    ("fc1 wgrad", f, h, T, False, False, True),
    ("qkv wgrad", 3 * h, h, T, False, False, True),
    ("lm wgrad", V, h, T, False, False, True),
    ("sq 8192", 8192, 8192, 8192, True, True, False),
]
for name, M, N, K, ak, bk, acc in cases:
    A = (torch.randn(M, K) if ak else torch.randn(K, M)).cuda().bfloat16()
    B = (torch.randn(N, K) if bk else torch.randn(K, N)).cuda().bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.float32 if acc else torch.bfloat16)
    from paper_2410_19367_b200.runtime.lib import OPT_GEMM_MODE, OPT_GEMM_WIDE
    res = []
    for mode, wide in ((1, 0), (2, 2), (2, 1)):
        ops.set_option(OPT_GEMM_MODE, mode)
        ops.set_option(OPT_GEMM_WIDE, wide)
        res.append(timeit(lambda: ops.gemm(A, B, C, a_kmajor=ak, b_kmajor=bk, beta=1.0 if acc else 0.0)))
    ops.set_option(OPT_GEMM_MODE, 0)
    ops.set_option(OPT_GEMM_WIDE, 0)
    ms1, ms, msw = res
    tfw = 2 * M * N * K / msw / 1e9
    opA = A if ak else A.t()
    opB = B.t() if bk else B
    ms_ref = timeit(lambda: torch.matmul(opA, opB))
    tf = 2 * M * N * K / ms / 1e9
    tf_ref = 2 * M * N * K / ms_ref / 1e9
    tf1 = 2 * M * N * K / ms1 / 1e9
    print(f"{name:12s} M={M:6d} N={N:6d} K={K:6d}  1sm {tf1:7.1f} | 2sm {ms*1e3:8.1f} us {tf:7.1f} TF/s | wide {tfw:7.1f} | cublas {ms_ref*1e3:8.1f} us {tf_ref:7.1f} TF/s | ratio {tf/tf_ref:.2f}", flush=True)
