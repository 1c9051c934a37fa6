"""Attention fwd/bwd timing: tcgen05 (impl 0) vs mma.sync flash (impl 2)."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import ops
from paper_2410_19367_b200.runtime.lib import OPT_ATTN_EXACT


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


for (B, S, H, Dh, causal) in [(1, 2048, 16, 128, True), (4, 512, 16, 64, False), (1, 2048, 32, 128, True)]:
    scale = 1 / math.sqrt(Dh)
    qkv = torch.randn(B * S, 3 * H * Dh, device="cuda").bfloat16()
    o = torch.empty(B * S, H * Dh, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda")
    dout = torch.randn_like(o)
    dqkv = torch.empty_like(qkv)
    ws = torch.empty(ops.attn_workspace_numel(B, S, H, Dh), device="cuda")
    f = 4.0 * B * H * S * S * Dh * (0.5 if causal else 1.0)
    line = f"B={B} S={S} H={H} Dh={Dh} causal={causal}:"
    for impl in (0, 2):
        ops.set_option(OPT_ATTN_EXACT, impl)
        tf = timeit(lambda: ops.attn_fwd(qkv, o, lse, B, S, H, Dh, causal, scale))
        tb = timeit(lambda: ops.attn_bwd(qkv, o, dout, lse, dqkv, ws, B, S, H, Dh, causal, scale))
        line += f" | {'tc' if impl == 0 else 'mma'} fwd {tf*1e3:7.1f} us {f/tf/1e9:6.1f} TF/s bwd {tb*1e3:7.1f} us {2.5*f/tb/1e9:6.1f} TF/s"
    ops.set_option(OPT_ATTN_EXACT, 0)
    print(line, flush=True)
