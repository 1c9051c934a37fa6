"""Per-iteration timestamps of the dK/dV softmax warp (CTA 0,0) from a
BP_ATTN_TRACE build (tools/libbitpipe_trace.so)."""
import ctypes
import math
import os
import sys

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import lib as L

L.LIB_PATH = os.path.abspath("tools/libbitpipe_trace.so")
import torch
from paper_2410_19367_b200.runtime import ops

B, S, H, Dh = 1, 2048, 16, 128
qkv = torch.randn(B * S, 3 * H * Dh, device="cuda").bfloat16()
o = torch.empty(B * S, H * Dh, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H * S, device="cuda")
dq = torch.empty_like(qkv)
ws = torch.empty(ops.attn_workspace_numel(B, S, H, Dh), device="cuda")
for _ in range(3):
    ops.attn_fwd(qkv, o, lse, B, S, H, Dh, True, 1 / math.sqrt(Dh))
    ops.attn_bwd(qkv, o, o, lse, dq, ws, B, S, H, Dh, True, 1 / math.sqrt(Dh))
torch.cuda.synchronize()
h = L.lib()
fn = h.bp_attn_trace_dump
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_longlong * 512)()
print("rc", fn(buf, 512))
t = [[buf[i * 8 + k] for k in range(8)] for i in range(64)]
base = t[0][0]
names = ["q_full wait", "sdp_full wait", "tmem ld", "compute", "mm_done wait", "st+arrive", "->next"]
print("iter  " + " ".join(f"{n:>13s}" for n in names))
for i in range(32):
    row = t[i]
    if row[0] == 0:
        break
    d = [row[k + 1] - row[k] for k in range(6)] + [(t[i + 1][0] - row[6]) if i + 1 < 64 and t[i + 1][0] else 0]
    print(f"{i:4d}  " + " ".join(f"{x:13d}" for x in d))
