"""Per-iteration timestamps of the dK/dV kernel (CTA 0,0) from a
BP_ATTN_TRACE build (tools/libbitpipe_trace.so): compute warp phases, the
MMA warp's issue points and the producer's Q-tile issue, all relative to the
compute warp's iteration start."""
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
from paper_2410_19367_b200.runtime.lib import OPT_ATTN_FWD_MODE
ops.set_option(OPT_ATTN_FWD_MODE, int(os.environ.get("FWD_MODE", "2")))  # trace the two-tile forward
for _ in range(3):
    ops.attn_fwd(qkv, o, lse, B, S, H, Dh, True, 1 / math.sqrt(Dh))
    ops.attn_bwd(qkv, o, o, lse, dq, ws, B, S, H, Dh, True, 1 / math.sqrt(Dh))
torch.cuda.synchronize()
h = L.lib()
fn = h.bp_attn_trace_dump
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_longlong * 1024)()
print("rc", fn(buf, 1024))
t = [[buf[i * 16 + k] for k in range(16)] for i in range(64)]
names = ["q_full", "sdp_full", "tmem_ld", "compute", "mm_done", "st+arr", "->next"]
print("iter " + " ".join(f"{n:>8s}" for n in names) + " | rel. to iter start: mma_top q_ok sdp_iss dvdk_iss prod_q")
for i in range(32):   # the traced thread (warp 4) is in compute group 0: even iterations only
    row = t[i]
    if row[0] == 0:
        continue
    nxt = t[i + 2][0] if i + 2 < 32 else 0
    d = [row[k + 1] - row[k] for k in range(6)] + [(nxt - row[6]) if nxt else 0]
    rel = [row[k] - row[0] if row[k] else 0 for k in (8, 9, 10, 11, 12)]
    print(f"{i:4d} " + " ".join(f"{x:8d}" for x in d) + " | " + " ".join(f"{x:8d}" for x in rel))

# forward (two-tile kernel), CTA (0,0) = last query-tile pair, rows 32..47;
# tile-A softmax warp (thread 96) phases, MMA issue points, producer loads
names = ["s_full", "max", "rescale", "exp+st", "arrive", "->next"]
print("fwd  " + " ".join(f"{n:>8s}" for n in names) + " | rel: PVA_p PVA_v S_A(j) PVB_p S_B(j) K(j) V(j)")
for j in range(16):
    row = t[32 + j]
    if row[0] == 0:
        break
    d = [row[k + 1] - row[k] for k in range(5)] + [(t[33 + j][0] - row[5]) if j < 15 and t[33 + j][0] else 0]
    rel = [row[k] - row[0] if row[k] else 0 for k in (8, 9, 10, 11, 12, 13, 14)]
    print(f"{j:4d} " + " ".join(f"{x:8d}" for x in d) + " | " + " ".join(f"{x:7d}" for x in rel))
