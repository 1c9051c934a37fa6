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
import os
pol = ps.paper_policy(D) if os.environ.get("ORDER", "paper") == "paper" else None
tr = Trainer(cfg, ps.build_bitpipe(D, N, policy=pol), dtype=torch.bfloat16, optim=OptimConfig(), record_timeline=True,
             partition=os.environ.get("PARTITION", "balanced"))
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

# time-weighted distribution of the number of tasks in flight (a task's span
# runs from its first kernel's start event to its end event on its stream)
ev = sorted([(a, 1) for a, b in spans] + [(b, -1) for a, b in spans])
hist, k, last = {}, 0, ev[0][0]
t0, t1 = ev[0][0], ev[-1][0]
edges = []
for t, dk in ev:
    hist[k] = hist.get(k, 0.0) + (t - last)
    edges.append((last, t, k))
    k += dk
    last = t
tot = t1 - t0
print("in-flight tasks: " + ", ".join(f"{kk}: {100 * v / tot:.1f}%" for kk, v in sorted(hist.items())))
for lo, hi in ((0.0, 0.1), (0.1, 0.9), (0.9, 1.0)):
    a, b = t0 + lo * tot, t0 + hi * tot
    w = sum(max(0.0, min(e, b) - max(s, a)) * kk for s, e, kk in edges)
    print(f"  mean in-flight over [{lo:.0%}, {hi:.0%}] of the step: {w / (b - a):.2f}")
