"""Do sub-wave tcgen05 GEMMs (64 CTA-pair tiles -> 128 of 148 SMs) overlap
across streams?  Times 2x20 launches of 2048x2048xK on one stream vs split
over two streams (and four)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import ops


def bufs(M, N, K):
    return (torch.randn(M, K, device="cuda").bfloat16(), torch.randn(N, K, device="cuda").bfloat16(),
            torch.empty(M, N, device="cuda", dtype=torch.bfloat16))


for K in (2048, 8192):
    sets = [bufs(2048, 2048, K) for _ in range(4)]
    streams = [torch.cuda.Stream() for _ in range(4)]
    n = 40

    def run(ns):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        evs = []
        for s in streams[:ns]:
            s.wait_event(e0)
        for i in range(n):
            j = i % ns
            A, B, C = sets[j]
            ops.gemm(A, B, C, stream=streams[j])
        for s in streams[:ns]:
            ev = torch.cuda.Event()
            ev.record(s)
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n * 1e3

    for ns in (1, 2, 4):
        run(ns)
    print(f"2048x2048x{K}: us/GEMM  1 stream {run(1):.1f} | 2 streams {run(2):.1f} | 4 streams {run(4):.1f}", flush=True)
