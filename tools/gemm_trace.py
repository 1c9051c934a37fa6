"""Per-CTA phase breakdown of single GEMM launches at the GPT-1.3B
micro-batch shapes, from the BP_GEMM_TRACE build (`make trace` ->
tools/libbitpipe_trace.so): prologue, wait for the first operand stage,
main loop, accumulator hand-off, epilogue, store drain, teardown (SM cycles,
median / max over the launch's CTAs), plus the spread of CTA start times
(global timer) and the launch's event time."""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import lib as L

L.LIB_PATH = os.path.abspath("tools/libbitpipe_trace.so")
import torch

from paper_2410_19367_b200.runtime import ops
from paper_2410_19367_b200.runtime.ops import EPI_GELU

h = 2048
dev = "cuda"
bf = torch.bfloat16
SHAPES = [  # name, M, N, K, kwargs builder
    ("proj fprop (bias+res)", 2048, h, h),
    ("qkv fprop (bias)", 2048, 3 * h, h),
    ("fc1 fprop (gelu)", 2048, 4 * h, h),
    ("fc2 fprop (bias+res)", 2048, h, 4 * h),
    ("fc1 dgrad (plain)", 2048, h, 4 * h),
    ("proj fprop (plain)", 2048, h, h),
    ("proj fprop (bias)", 2048, h, h),
    ("proj fprop (res)", 2048, h, h),
]
lib = L.lib()
dump = lib.bp_gemm_trace_dump
dump.argtypes = [ctypes.c_void_p, ctypes.c_int]
names = ["prologue", "1st stage", "mainloop", "acc->epi", "epilogue", "drain", "teardown"]
print(f"{'shape':24s} {'ms/launch':>9s} {'CTAs':>5s} {'tiles':>5s} {'start spread us':>15s} | "
      + " ".join(f"{n:>10s}" for n in names) + "   (median cycles; max in brackets)")
for name, M, N, K in SHAPES:
    a = torch.randn(M, K, device=dev).to(bf)
    dgrad = "dgrad" in name
    w = (torch.randn(K, N, device=dev) if dgrad else torch.randn(N, K, device=dev)).to(bf) * 0.02
    c = torch.empty(M, N, device=dev, dtype=bf)
    bias = torch.randn(N, device=dev).to(bf)
    kw = {} if ("plain" in name or name.endswith("(res)")) else {"bias": bias}
    if dgrad:
        kw["b_kmajor"] = False
    if "res" in name:
        kw["residual"] = torch.randn(M, N, device=dev).to(bf)
    if "gelu" in name:
        kw["aux"] = torch.empty_like(c)
        kw["epilogue"] = EPI_GELU
    for _ in range(5):
        ops.gemm(a, w, c, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        ops.gemm(a, w, c, **kw)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    torch.cuda.synchronize()
    NB = 320 * 10 + 320 * 8 * 5
    buf = (ctypes.c_longlong * NB)()
    assert dump(buf, NB) == 0
    rows = [[buf[i * 10 + k] for k in range(10)] for i in range(320)]
    rows = [r for r in rows if r[0]]
    lead = [r for i, r in enumerate(rows) if r[2]]  # leader CTAs carry the MMA stamps
    g0 = min(r[8] for r in rows)
    spread = (max(r[8] for r in rows) - g0) / 1e3
    ph = {n: [] for n in names}
    for r in lead:
        ph["prologue"].append(r[1] - r[0])
        ph["1st stage"].append(r[2] - r[1])
        ph["mainloop"].append(r[3] - r[2])
        ph["acc->epi"].append(r[4] - r[3])
        ph["epilogue"].append(r[5] - r[4])
        ph["drain"].append(r[6] - r[5])
        ph["teardown"].append(r[7] - r[6])
    tiles = statistics.median(r[9] for r in rows)
    cells = " ".join(f"{int(statistics.median(v)):>5d}[{max(v):>5d}]".rjust(10) if v else "-" for v in ph.values())
    print(f"{name:24s} {ms * 1e3:8.1f}u {len(rows):5d} {tiles:5.0f} {spread:15.2f} | {cells}")
    # per-chunk epilogue stamps (first tile, epilogue warp 0) of CTA 0:
    # tmem ld, input wait, store-slot wait + staging, store issue, -> next chunk
    base = 320 * 10
    ch = [[buf[base + (0 * 8 + c) * 5 + k] for k in range(5)] for c in range(8)]
    parts = []
    for c in range(8):
        t = ch[c]
        if not t[0]:
            break
        nxt = ch[c + 1][0] if c + 1 < 8 and ch[c + 1][0] else t[4]
        parts.append(f"c{c}: ld {t[1] - t[0]} in {t[2] - t[1] if t[2] else 0} st {t[3] - (t[2] or t[1])} "
                     f"iss {t[4] - t[3]} nx {nxt - t[4]}")
    print("    epilogue chunks (cycles): " + " | ".join(parts))
