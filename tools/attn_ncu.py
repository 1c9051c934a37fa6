"""One launch each of the causal attention kernels at the GPT-1.3B shape
(B=1, S=2048, H=16, Dh=128) after warm-up, for `ncu --set full -k
regex:"fwd_tc|dkdv_tc|dq_ds_tc" --launch-skip 6 --launch-count 3`."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import ops

B, S, H, Dh = 1, 2048, 16, 128
qkv = torch.randn(B * S, 3 * H * Dh, device="cuda").bfloat16()
o = torch.empty(B * S, H * Dh, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H * S, device="cuda")
dout = torch.randn_like(o)
dqkv = torch.empty_like(qkv)
ws = torch.empty(ops.attn_workspace_numel(B, S, H, Dh), device="cuda")
for _ in range(3):
    ops.attn_fwd(qkv, o, lse, B, S, H, Dh, True, 1 / math.sqrt(Dh))
    ops.attn_bwd(qkv, o, dout, lse, dqkv, ws, B, S, H, Dh, True, 1 / math.sqrt(Dh))
torch.cuda.synchronize()
