"""Per-launch time of the 2-SM tcgen05 GEMM at each forced pair-tile width
(BP_OPT_GEMM_BN) on the GPT-1.3B / BERT-large per-micro-batch shapes, with
the real epilogues (bias, residual, GELU), L2 flushed between launches."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import ops
from paper_2410_19367_b200.runtime.lib import EPI_GELU, OPT_GEMM_BN

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
    bb = torch.randn(N, device="cuda").bfloat16() if bias else None
    rr = torch.randn(M, N, device="cuda").bfloat16() if res else None
    aux = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if gelu else None
    kw = dict(b_kmajor=bk, bias=bb, residual=rr)
    if gelu:
        kw.update(aux=aux, epilogue=EPI_GELU)
    out = []
    for bn in (0, 256, 224, 192, 128):
        ops.set_option(OPT_GEMM_BN, bn)
        ms = timeit(lambda: ops.gemm(A, B, C, **kw))
        out.append(f"{'auto' if bn == 0 else bn}: {ms * 1e3:6.1f} us {2 * M * N * K / ms / 1e9:6.0f} TF/s")
    ops.set_option(OPT_GEMM_BN, 0)
    print(f"{name:22s} {M}x{N}x{K} | " + " | ".join(out), flush=True)


T, h = 2048, 2048
case("qkv fprop (bias)", T, 3 * h, h, bias=True)
case("proj fprop (bias+res)", T, h, h, bias=True, res=True)
case("fc1 fprop (bias+gelu)", T, 4 * h, h, bias=True, gelu=True)
case("fc2 fprop (bias+res)", T, h, 4 * h, bias=True, res=True)
case("proj dgrad", T, h, h, bk=False)
case("qkv dgrad", T, h, 3 * h, bk=False)
case("fc1 dgrad", T, h, 4 * h, bk=False)
case("fc2 dgrad", T, 4 * h, h, bk=False)
h = 1024
case("bert qkv fprop", T, 3 * h, h, bias=True)
case("bert proj fprop", T, h, h, bias=True, res=True)
case("bert fc2 fprop", T, h, 4 * h, bias=True, res=True)
