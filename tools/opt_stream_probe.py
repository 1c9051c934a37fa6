import sys, time, torch
sys.path.insert(0, ".")
from paper_2410_19367_b200 import schedule as ps
from paper_2410_19367_b200.model import CONFIGS, synthetic_batch
from paper_2410_19367_b200.runtime.executor import Trainer
cfg = CONFIGS["gpt-1.3b"]
tr = Trainer(cfg, ps.build_bitpipe(8, 16, 2), dtype=torch.bfloat16, partition="balanced")
tok, tgt = synthetic_batch(cfg, 16)
tok, tgt = tok.int().cuda(), tgt.int().cuda()
for i in range(8):
    t0 = time.time()
    tr.train_step(tok, tgt); torch.cuda.synchronize()
    print(i, round((time.time() - t0) * 1e3, 1), "ms", flush=True)
