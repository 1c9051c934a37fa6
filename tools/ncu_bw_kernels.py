"""One launch each of the HBM-bound kernels at GPT-1.3B shapes (LayerNorm
fwd / bwd 2048x2048, softmax cross-entropy 2048x50304, AdamW over one
stage's ~88 M parameters, embedding fwd / bwd), after a warm-up launch, for
`ncu --set full` (achieved DRAM GB/s vs peak)."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import ops

M, h, V = 2048, 2048, 50304
x = torch.randn(M, h, device="cuda").bfloat16()
g = torch.ones(h, device="cuda").bfloat16()
b = torch.zeros(h, device="cuda").bfloat16()
y = torch.empty_like(x)
mean = torch.empty(M, device="cuda")
rstd = torch.empty(M, device="cuda")
dy, dres, dx = torch.randn_like(x), torch.randn_like(x), torch.empty_like(x)
dg, db, cs = (torch.zeros(h, device="cuda") for _ in range(3))
logits = torch.randn(M, V, device="cuda").bfloat16()
tgt = torch.randint(0, V, (M,), device="cuda", dtype=torch.int32)
loss = torch.zeros(1, device="cuda")
n = 88 * 1024 * 1024
master, ga, gb_, m, v = (torch.randn(n, device="cuda") for _ in range(5))
pa = torch.empty(n, device="cuda", dtype=torch.bfloat16)
pb = torch.empty_like(pa)
wte = torch.randn(V, h, device="cuda").bfloat16()
wpe = torch.randn(M, h, device="cuda").bfloat16()
tok = torch.randint(0, V, (M,), device="cuda", dtype=torch.int32)
dwte = torch.zeros(V, h, device="cuda")
dwpe = torch.zeros(M, h, device="cuda")


def run():
    ops.layernorm_fwd(x, g, b, y, mean, rstd)
    ops.layernorm_bwd(dy, x, g, mean, rstd, dx, dg, db, dres=dres, dx_colsum=cs)
    ops.xent_fwd_bwd(logits, tgt, loss, grad_scale=1.0 / M, loss_scale=1.0 / M)
    ops.adam(master, ga, gb_, m, v, pa, pb, lr=1e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1, step=1)
    ops.embed_fwd(tok, wte, wpe, y, 1, M)
    ops.embed_bwd(tok, dy, dwte, dwpe, 1, M)


run()
torch.cuda.synchronize()
run()
torch.cuda.synchronize()
print("done")
