"""Run warm-up steps, then one profiled train step between
cudaProfilerStart/Stop (use with ncu --profile-from-start off)."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200 import schedule as ps
from paper_2410_19367_b200.model import CONFIGS, OptimConfig, synthetic_batch
from paper_2410_19367_b200.runtime.executor import Trainer

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="gpt-1.3b")
ap.add_argument("--D", type=int, default=8)
ap.add_argument("--N", type=int, default=16)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--order", default="paper", choices=["paper", "search"])
ap.add_argument("--partition", default="auto")
args = ap.parse_args()
cfg = CONFIGS[args.config]
# the bench's configuration: F2 paper-policy order, its default partition ("auto")
sched = ps.build_bitpipe(args.D, args.N, policy=ps.search_bitpipe_policy(args.D, args.N)[0]
                         if args.order == "search" else ps.paper_policy(args.D))
tr = Trainer(cfg, sched, dtype=torch.bfloat16, optim=OptimConfig(), partition=args.partition)
tok, tgt = synthetic_batch(cfg, args.N)
tok, tgt = tok.int().cuda(), tgt.int().cuda()
for _ in range(args.warmup):
    tr.train_step(tok, tgt)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
tr.train_step(tok, tgt)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("profiled one step")
