"""One launch each of the GPT-1.3B GEMM classes (after warm-up), for
`ncu --set full -k regex:gemm_tc2 --launch-skip 5`: fc1 fprop, fc2 fprop,
fc1 dgrad, fc1 wgrad, qkv fprop."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import ops

T, h, f = 2048, 2048, 8192
cases = [("fc1 fprop", T, f, h, True, True, False), ("fc2 fprop", T, h, f, True, True, False),
         ("fc1 dgrad", T, h, f, True, False, False), ("fc1 wgrad", f, h, T, False, False, True),
         ("qkv fprop", T, 3 * h, h, True, True, False)]
bufs = []
for name, M, N, K, ak, bk, acc in cases:
    A = (torch.randn(M, K) if ak else torch.randn(K, M)).cuda().bfloat16()
    B = (torch.randn(N, K) if bk else torch.randn(K, N)).cuda().bfloat16()
    C = torch.zeros(M, N, device="cuda", dtype=torch.float32 if acc else torch.bfloat16)
    bufs.append((A, B, C, ak, bk, acc))
for A, B, C, ak, bk, acc in bufs:  # warm-up: 5 launches
    ops.gemm(A, B, C, a_kmajor=ak, b_kmajor=bk, beta=1.0 if acc else 0.0)
for A, B, C, ak, bk, acc in bufs:  # profiled
    ops.gemm(A, B, C, a_kmajor=ak, b_kmajor=bk, beta=1.0 if acc else 0.0)
torch.cuda.synchronize()
print("done")
