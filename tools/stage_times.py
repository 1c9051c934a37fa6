"""Isolated per-stage forward / backward device times of the GPT-1.3B
BitPipe D=8 stages (Trainer.measure_task_times) -- calibration data for the
partition cost model.  Prints one line per (direction, stage)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200 import schedule as ps
from paper_2410_19367_b200.model import CONFIGS
from paper_2410_19367_b200.runtime.executor import Trainer

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "gpt-1.3b"]
part = sys.argv[2] if len(sys.argv) > 2 else "uniform"
tr = Trainer(cfg, ps.build_bitpipe(8, 16), dtype=torch.bfloat16, partition=part)
times = tr.measure_task_times()
rows = []
for (dr, s, k), ms in sorted(times.items(), key=lambda x: (str(x[0][0]), x[0][1], x[0][2])):
    rows.append({"dir": str(dr), "stage": s, "kind": k, "ms": ms, "hb": list(tr.plans[s].halfblocks)})
print(json.dumps({"partition": tr.partition, "rows": rows}))
