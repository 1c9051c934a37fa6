"""1-SM (BM = 128) vs 2-SM (CTA pair, BM = 256) tcgen05 GEMM per-launch time
on the per-micro-batch shapes (L2 flushed between launches)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import ops
from paper_2410_19367_b200.runtime.lib import EPI_GELU, OPT_GEMM_MODE

flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def case(name, M, N, K, bk=True, bias=False, res=False, gelu=False):
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(N, K) if bk else torch.randn(K, N)).cuda().bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    kw = dict(b_kmajor=bk, bias=torch.randn(N, device="cuda").bfloat16() if bias else None,
              residual=torch.randn(M, N, device="cuda").bfloat16() if res else None)
    if gelu:
        kw.update(aux=torch.empty(M, N, device="cuda", dtype=torch.bfloat16), epilogue=EPI_GELU)
    out = []
    for mode in (1, 2):
        ops.set_option(OPT_GEMM_MODE, mode)
        ms = timeit(lambda: ops.gemm(A, B, C, **kw))
        out.append(f"{'1sm' if mode == 1 else '2sm'}: {ms * 1e3:6.1f} us {2 * M * N * K / ms / 1e9:6.0f} TF/s")
    ops.set_option(OPT_GEMM_MODE, 0)
    print(f"{name:24s} {M}x{N}x{K} | " + " | ".join(out), flush=True)


T = 2048
for h in (1024, 2048):
    case(f"h{h} qkv fprop (bias)", T, 3 * h, h, bias=True)
    case(f"h{h} proj fprop (b+res)", T, h, h, bias=True, res=True)
    case(f"h{h} fc1 fprop (b+gelu)", T, 4 * h, h, bias=True, gelu=True)
    case(f"h{h} fc2 fprop (b+res)", T, h, 4 * h, bias=True, res=True)
    case(f"h{h} proj dgrad", T, h, h, bk=False)
    case(f"h{h} qkv dgrad", T, h, 3 * h, bk=False)
    case(f"h{h} fc1 dgrad", T, h, 4 * h, bk=False)
    case(f"h{h} fc2 dgrad", T, 4 * h, h, bk=False)
