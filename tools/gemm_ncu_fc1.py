"""The fc1 forward GEMM exactly as the co-resident step issues it (2048 x
8192 x 2048, bias + GELU with the saved pre-activation, throughput tile pick,
L2 hints on), for `ncu --set full -k regex:gemm_tc2 --launch-skip 3
--launch-count 3`: the DRAM bytes per launch are bench.py's roofline
`traffic`."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import lib as L
from paper_2410_19367_b200.runtime import ops

T, h, f = 2048, 2048, 8192
ops.set_option(L.OPT_GEMM_PICK, 1)
X = torch.randn(T, h, device="cuda").bfloat16()
W = (torch.randn(f, h, device="cuda") * 0.02).bfloat16()
b = torch.randn(f, device="cuda").bfloat16()
Y = torch.empty(T, f, device="cuda", dtype=torch.bfloat16)
pre = torch.empty_like(Y)
for _ in range(6):
    ops.gemm(X, W, Y, bias=b, aux=pre, epilogue=L.EPI_GELU)
torch.cuda.synchronize()
