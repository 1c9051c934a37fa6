"""Per-iteration timestamps (SM cycles) of the one-query-tile causal
attention forward (fwd_tc), CTA (0, 0) = the heaviest query tile (16 key
tiles at S = 2048), from a BP_ATTN_TRACE build (make trace ->
tools/libbitpipe_trace.so).  Softmax warp 4 lane 0 phases per key tile j:
wait for S(j), TMEM load (+ s_free arrive), row max + half exchange,
rescale, exponentials, pack, P store + arrive; then the MMA warp's issue
points of S(j) / P V(j) and the producer's K(j) issue, relative to the
softmax's start of tile j."""
import ctypes
import math
import os
import sys

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import lib as L

L.LIB_PATH = os.path.abspath("tools/libbitpipe_trace.so")
import torch
from paper_2410_19367_b200.runtime import ops
from paper_2410_19367_b200.runtime.lib import OPT_ATTN_FWD_MODE

B, S, H, Dh = 1, 2048, int(os.environ.get("H", "16")), 128
qkv = torch.randn(B * S, 3 * H * Dh, device="cuda").bfloat16()
o = torch.empty(B * S, H * Dh, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H * S, device="cuda")
ops.set_option(OPT_ATTN_FWD_MODE, 1)
for _ in range(3):
    ops.attn_fwd(qkv, o, lse, B, S, H, Dh, True, 1 / math.sqrt(Dh))
torch.cuda.synchronize()
h = L.lib()
fn = h.bp_attn_trace_dump
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_longlong * 1024)()
fn(buf, 1024)
t = [[buf[i * 16 + k] for k in range(16)] for i in range(64)]
names = ["wait_S", "tmem_ld", "max+xchg", "rescale", "exp", "pack", "st+arr", "->next"]
print("j    " + " ".join(f"{n:>8s}" for n in names) + " | rel: S_iss PV_iss K_iss S_top S_kok PV_top PV_pok PV_mmas")
tot = 0
for j in range(16):
    row = t[32 + j]
    if row[0] == 0:
        break
    nxt = t[33 + j][0] if j < 15 else 0
    d = [row[k + 1] - row[k] for k in range(7)] + [(nxt - row[7]) if nxt else 0]
    rel = [row[k] - row[0] if row[k] else 0 for k in (8, 9, 10, 11, 12, 13, 14, 15)]
    if nxt:
        tot += nxt - row[0]
    print(f"{j:4d} " + " ".join(f"{x:8d}" for x in d) + " | " + " ".join(f"{x:7d}" for x in rel))
print("mean tile period (cycles):", tot / 15)
