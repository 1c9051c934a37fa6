"""A/B of the attention forward's FMA-pipe exponential fraction
(BP_OPT_ATTN_FWD_EXF = 2..5 of every 8): time (interleaved rounds, min) and
the max |O| difference against the default."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import lib as L
from paper_2410_19367_b200.runtime import ops


def timeit(fn, iters=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / iters


for (B, S, H, Dh, causal) in [(1, 2048, 16, 128, True), (1, 2048, 32, 128, True), (4, 512, 16, 64, False)]:
    scale = 1 / math.sqrt(Dh)
    qkv = torch.randn(B * S, 3 * H * Dh, device="cuda").bfloat16()
    o = torch.empty(B * S, H * Dh, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda")
    ops.set_option(L.OPT_ATTN_FWD_MODE, 1)
    ref = None
    res = {}
    for rnd in range(3):
        for exf in (2, 6):
            ops.set_option(L.OPT_ATTN_FWD_EXF, exf)
            ops.attn_fwd(qkv, o, lse, B, S, H, Dh, causal, scale)
            torch.cuda.synchronize()
            if rnd == 0:
                if exf == 2:
                    ref = o.float().clone()
                d = (o.float() - ref).abs().max().item()
                res[exf] = [d, []]
            res[exf][1].append(timeit(lambda: ops.attn_fwd(qkv, o, lse, B, S, H, Dh, causal, scale)))
    f = 4.0 * B * H * S * S * Dh * (0.5 if causal else 1.0)
    print(f"B={B} S={S} H={H} Dh={Dh} causal={causal}: " + " | ".join(
        f"exf {k}: {min(v[1]):6.1f} us {f / min(v[1]) / 1e6:5.0f} TF/s (max|dO| {v[0]:.1e})" for k, v in res.items()),
        flush=True)
    ops.set_option(L.OPT_ATTN_FWD_EXF, 0)
    ops.set_option(L.OPT_ATTN_FWD_MODE, 0)
