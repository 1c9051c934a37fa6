"""Is the co-resident train step host-bound?  Compares the host time to
enqueue one GPT-1.3B BitPipe step (D=8, N=16) with its device time."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200 import schedule as ps
from paper_2410_19367_b200.model import CONFIGS, synthetic_batch
from paper_2410_19367_b200.runtime import ops
from paper_2410_19367_b200.runtime.executor import Trainer

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "gpt-1.3b"]
D, N = 8, 16
tr = Trainer(cfg, ps.build_bitpipe(D, N, 2), dtype=torch.bfloat16)
tok, tgt = synthetic_batch(cfg, N)
tok, tgt = tok.int().cuda(), tgt.int().cuda()
for _ in range(3):
    tr.train_step(tok, tgt)
torch.cuda.synchronize()
for _ in range(3):
    l0 = ops.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    tr.train_step(tok, tgt)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"enqueue {1e3*(t1-t0):.1f} ms  wall {1e3*(t2-t0):.1f} ms  device {e0.elapsed_time(e1):.1f} ms  "
          f"launches {ops.launch_count()-l0}  host us/launch {1e6*(t1-t0)/(ops.launch_count()-l0):.1f}", flush=True)
