"""fc1-forward GEMM (2048x8192x2048) with L2-hot operands (same buffers every
launch) vs L2-cold operands (rotating through > 126 MB of buffer sets), and
the same for the wgrad shape.  Separates operand-fetch effects from the
kernel's mainloop."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import ops


def run(M, N, K, ak, bk, acc, nsets, iters=40):
    sets = []
    for _ in range(nsets):
        A = (torch.randn(M, K) if ak else torch.randn(K, M)).cuda().bfloat16()
        B = (torch.randn(N, K) if bk else torch.randn(K, N)).cuda().bfloat16()
        C = torch.zeros(M, N, device="cuda", dtype=torch.float32 if acc else torch.bfloat16)
        sets.append((A, B, C))
    for i in range(3):
        A, B, C = sets[i % nsets]
        ops.gemm(A, B, C, a_kmajor=ak, b_kmajor=bk, beta=1.0 if acc else 0.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        A, B, C = sets[i % nsets]
        ops.gemm(A, B, C, a_kmajor=ak, b_kmajor=bk, beta=1.0 if acc else 0.0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    return ms, 2.0 * M * N * K / ms / 1e9


for name, M, N, K, ak, bk, acc in [("fc1 fprop", 2048, 8192, 2048, True, True, False),
                                    ("fc1 wgrad", 8192, 2048, 2048, False, False, True),
                                    ("proj fprop", 2048, 2048, 2048, True, True, False)]:
    hot = run(M, N, K, ak, bk, acc, 1)
    cold = run(M, N, K, ak, bk, acc, 8)
    print(f"{name:10s} hot {hot[0]*1e3:7.1f} us {hot[1]:7.1f} TF/s | cold(8 sets) {cold[0]*1e3:7.1f} us {cold[1]:7.1f} TF/s",
          flush=True)
