"""Tiny driver for `ncu --set full`: one fc1-forward GEMM (the bench's
roofline kernel) and one causal attention fwd/bwd at GPT-1.3B shapes."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import ops

M, H, F = 2048, 2048, 8192
A = torch.randn(M, H, device="cuda").bfloat16()
W = torch.randn(F, H, device="cuda").bfloat16()
C = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    ops.gemm(A, W, C)
B, S, NH, Dh = 1, 2048, 16, 128
qkv = torch.randn(B * S, 3 * NH * Dh, device="cuda").bfloat16()
o = torch.empty(B * S, NH * Dh, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * NH * S, device="cuda")
dq = torch.empty_like(qkv)
ws = torch.empty(ops.attn_workspace_numel(B, S, NH, Dh), device="cuda")
for _ in range(2):
    ops.attn_fwd(qkv, o, lse, B, S, NH, Dh, True, 1 / math.sqrt(Dh))
    ops.attn_bwd(qkv, o, o, lse, dq, ws, B, S, NH, Dh, True, 1 / math.sqrt(Dh))
torch.cuda.synchronize()
print("done")
