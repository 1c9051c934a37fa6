"""A/B device time of the GPT-1.3B BitPipe step (D=8, N=16, one GPU) under
library option settings: `python tools/ab_step.py OPT=VAL[,OPT=VAL] ...`;
each argument is one variant (`base` = defaults).  Variants are interleaved
over several rounds so clock drift hits all of them alike."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200 import schedule as ps
from paper_2410_19367_b200.model import CONFIGS, synthetic_batch
from paper_2410_19367_b200.runtime import lib as L
from paper_2410_19367_b200.runtime import ops
from paper_2410_19367_b200.runtime.executor import Trainer

variants = sys.argv[1:] or ["base"]
cfg = CONFIGS["gpt-1.3b"]
tr = Trainer(cfg, ps.build_bitpipe(8, 16, 2), dtype=torch.bfloat16)
tok, tgt = synthetic_batch(cfg, 16)
tok, tgt = tok.int().cuda(), tgt.int().cuda()


def apply(v, reset=False):
    if v == "base":
        return
    for kv in v.split(","):
        k, val = kv.split("=")
        defaults = {"OPT_STREAM_K": 2, "OPT_GEMM_L2_HINTS": 1, "OPT_LN_CTAS_PER_SM": 1}
        ops.set_option(getattr(L, k), defaults.get(k, 0) if reset else int(val))


for _ in range(3):
    tr.train_step(tok, tgt)
res = {v: [] for v in variants}
for rnd in range(3):
    for v in variants:
        apply(v)
        tr.train_step(tok, tgt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            tr.train_step(tok, tgt)
        e1.record()
        torch.cuda.synchronize()
        res[v].append(e0.elapsed_time(e1) / 3)
        apply(v, reset=True)
for v in variants:
    print(f"{v:40s} ms/step " + " ".join(f"{t:7.1f}" for t in res[v]) + f"  min {min(res[v]):.1f}", flush=True)
