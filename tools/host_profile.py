"""Where the host time of one eager co-resident train step goes (cProfile,
sorted by own time): `python tools/host_profile.py [config]`."""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200 import schedule as ps
from paper_2410_19367_b200.model import CONFIGS, synthetic_batch
from paper_2410_19367_b200.runtime.executor import Trainer

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "gpt-1.3b"]
D, N = (4, 8) if cfg.name == "bert-large" else (8, 16)
tr = Trainer(cfg, ps.build_bitpipe(D, N, 2), dtype=torch.bfloat16)
tok, tgt = synthetic_batch(cfg, N)
tok, tgt = tok.int().cuda(), tgt.int().cuda()
for _ in range(3):
    tr.train_step(tok, tgt)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(2):
    tr.train_step(tok, tgt)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
