"""Bitwise comparison of the attention forward and backward between two builds:
`python tools/attn_bitwise.py save LIB OUT` then `... check LIB OUT`."""
import math
import os
import sys

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import lib as L

mode, libp, out = sys.argv[1], sys.argv[2], sys.argv[3]
L.LIB_PATH = os.path.abspath(libp)
import torch
from paper_2410_19367_b200.runtime import ops

torch.manual_seed(0)
res = {}
for (B, S, H, Dh, causal) in [(1, 2048, 16, 128, True), (4, 512, 16, 64, False), (2, 1024, 8, 128, False)]:
    qkv = (torch.randn(B * S, 3 * H * Dh, device="cuda") * 2).bfloat16()
    o = torch.empty(B * S, H * Dh, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda")
    ops.attn_fwd(qkv, o, lse, B, S, H, Dh, causal, 1 / math.sqrt(Dh))
    dout = torch.randn_like(o)
    dqkv = torch.empty_like(qkv)
    ws = torch.empty(ops.attn_workspace_numel(B, S, H, Dh), device="cuda")
    ops.attn_bwd(qkv, o, dout, lse, dqkv, ws, B, S, H, Dh, causal, 1 / math.sqrt(Dh))
    torch.cuda.synchronize()
    res[(B, S, H, Dh, causal)] = (o.cpu(), lse.cpu(), dqkv.cpu())
if mode == "save":
    torch.save(res, out)
else:
    ref = torch.load(out)
    for k, (o, lse, dq) in res.items():
        o0, l0, dq0 = ref[k]
        print(k, "O bit-identical" if torch.equal(o.view(torch.int16), o0.view(torch.int16)) else
              f"O differs: {(o.view(torch.int16) != o0.view(torch.int16)).sum().item()} elements, "
              f"max {(o.float() - o0.float()).abs().max().item():.3g}",
              "| lse bit-identical" if torch.equal(lse.view(torch.int32), l0.view(torch.int32)) else
              f"| lse differs max {(lse - l0).abs().max().item():.3g}",
              "| dQKV bit-identical" if torch.equal(dq.view(torch.int16), dq0.view(torch.int16)) else
              f"| dQKV differs: {(dq.view(torch.int16) != dq0.view(torch.int16)).sum().item()} elements")
