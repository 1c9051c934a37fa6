"""One vs two query-tile forward kernels (BP_OPT_ATTN_FWD_MODE 1 / 2) on
the GPT-1.3B / BERT-large attention shapes; BP_LIB=path times another build."""
import math, os, sys
sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import lib as L
if os.environ.get("BP_LIB"):
    L.LIB_PATH = os.path.abspath(os.environ["BP_LIB"])
import torch
from paper_2410_19367_b200.runtime import ops
def timeit(fn, iters=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / iters
for (B, S, H, Dh, causal) in [(1, 2048, 16, 128, False), (1, 2048, 16, 128, True), (1, 4096, 16, 128, False), (4, 512, 16, 64, False)]:
    qkv = torch.randn(B * S, 3 * H * Dh, device="cuda").bfloat16()
    o = torch.empty(B * S, H * Dh, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda")
    f = 4.0 * B * H * S * S * Dh * (0.5 if causal else 1.0)
    r = []
    for m in (1, 2):
        ops.set_option(L.OPT_ATTN_FWD_MODE, m)
        t = timeit(lambda: ops.attn_fwd(qkv, o, lse, B, S, H, Dh, causal, 1 / math.sqrt(Dh)))
        r.append(f"mode {m}: {t:6.1f} us {f / t / 1e6:5.0f} TF/s")
    print(B, S, H, Dh, causal, " | ".join(r), flush=True)
