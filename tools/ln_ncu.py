"""ncu driver: one fused LayerNorm backward at 2048 x 2048 bf16."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import ops

rows, cols = 2048, 2048
x = torch.randn(rows, cols, device="cuda").bfloat16()
g = torch.randn(cols, device="cuda").bfloat16()
b = torch.randn(cols, device="cuda").bfloat16()
y = torch.empty_like(x)
mean = torch.empty(rows, device="cuda")
rstd = torch.empty(rows, device="cuda")
dy, dres, dx = torch.randn_like(x), torch.randn_like(x), torch.empty_like(x)
dg, db, cs = (torch.zeros(cols, device="cuda") for _ in range(3))
ops.layernorm_fwd(x, g, b, y, mean, rstd)
for _ in range(3):
    ops.layernorm_bwd(dy, x, g, mean, rstd, dx, dg, db, dres=dres, dx_colsum=cs)
torch.cuda.synchronize()
