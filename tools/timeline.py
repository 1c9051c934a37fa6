"""Per-task CUDA-event timeline of one co-resident train step: how much do
the D logical-device streams overlap on the single GPU?"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200 import schedule as ps
from paper_2410_19367_b200.model import CONFIGS, OptimConfig, synthetic_batch
from paper_2410_19367_b200.runtime.executor import Trainer

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "gpt-1.3b"]
D, N = 8, 16
tr = Trainer(cfg, ps.build_bitpipe(D, N), dtype=torch.bfloat16, optim=OptimConfig(), record_timeline=True)
tok, tgt = synthetic_batch(cfg, N)
tok, tgt = tok.int().cuda(), tgt.int().cuda()
import time
for _ in range(3):
    t0 = time.perf_counter()
    tr.train_step(tok, tgt)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host issue {1e3*(t1-t0):.1f} ms, wall incl. sync {1e3*(t2-t0):.1f} ms")
info = tr.measured_bubble()
tl = tr.timeline
first = tl[0][2]
spans = sorted((first.elapsed_time(e0), first.elapsed_time(e1)) for d, t, e0, e1 in tl)
busy_sum = sum(b - a for a, b in spans)
# union of intervals = time at least one task is running
union, cur_a, cur_b = 0.0, None, None
for a, b in spans:
    if cur_b is None or a > cur_b:
        if cur_b is not None:
            union += cur_b - cur_a
        cur_a, cur_b = a, b
    else:
        cur_b = max(cur_b, b)
union += cur_b - cur_a
print(f"makespan {info['makespan_ms']:.1f} ms; sum of task spans {busy_sum:.1f} ms; union {union:.1f} ms; "
      f"mean concurrency {busy_sum / union:.2f}; per-device busy ms {[round(v, 1) for v in info['busy_ms'].values()]}")
