"""proj fprop (2048 x 2048 x 2048, bias + residual: one tile per CTA pair)
with 4 then 8 epilogue warps, for `ncu --set full -k regex:gemm_tc2
--launch-skip 4 --launch-count 2` (4 warm-up launches, then EW=4, EW=8)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import lib as L
from paper_2410_19367_b200.runtime import ops

T = h = 2048
X = torch.randn(T, h, device="cuda").bfloat16()
W = (torch.randn(h, h, device="cuda") * 0.02).bfloat16()
b = torch.randn(h, device="cuda").bfloat16()
R = torch.randn(T, h, device="cuda").bfloat16()
C = torch.empty(T, h, device="cuda", dtype=torch.bfloat16)
for ew in (4, 8, 4, 8, 4, 8):
    ops.set_option(L.OPT_GEMM_EPI_WARPS, ew)
    ops.gemm(X, W, C, bias=b, residual=R)
torch.cuda.synchronize()
