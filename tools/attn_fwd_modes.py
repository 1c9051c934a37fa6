"""Forward attention time per kernel variant (OPT_ATTN_FWD_MODE 1 = one
query tile per CTA, 2 = two tiles) at the BASELINE shapes."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import ops
from paper_2410_19367_b200.runtime.lib import OPT_ATTN_FWD_MODE


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
    return s.elapsed_time(e) / iters * 1e3


for (B, S, H, Dh, c) in [(1, 2048, 16, 128, True), (1, 2048, 32, 128, True), (4, 512, 16, 64, False),
                         (2, 2048, 16, 128, True)]:
    qkv = torch.randn(B * S, 3 * H * Dh, device="cuda").bfloat16()
    o = torch.empty(B * S, H * Dh, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda")
    res = []
    for mode in (1, 2):
        ops.set_option(OPT_ATTN_FWD_MODE, mode)
        res.append(timeit(lambda: ops.attn_fwd(qkv, o, lse, B, S, H, Dh, c, 1 / math.sqrt(Dh))))
    ops.set_option(OPT_ATTN_FWD_MODE, 0)
    print(f"B={B} S={S} H={H} Dh={Dh} causal={c}: 1-tile {res[0]:.1f} us, 2-tile {res[1]:.1f} us", flush=True)
