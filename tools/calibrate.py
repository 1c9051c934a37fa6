"""Fit the partitioner's measured cost table (model.fit_task_costs) from one
or more bench runs' task times and write
paper_2410_19367_b200/calibration/<config>.json.

  python bench.py [--config C] --dump-task-times tt.json          (on the B200)
  python tools/calibrate.py "<provenance>" tt1.json [tt2.json ...]  (anywhere)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_19367_b200.model import CONFIGS, fit_task_costs  # noqa: E402
from paper_2410_19367_b200.schedule import Direction  # noqa: E402

runs = [json.load(open(f)) for f in sys.argv[2:]]
names = {next(k for k, c in CONFIGS.items() if c.name == r["config"]) for r in runs}
assert len(names) == 1, f"runs of different configs: {names}"
name = names.pop()
data = [(r["partition"], {(Direction(dr), s, k): v for dr, s, k, v in r["times"]}, r["N"] // 2) for r in runs]
costs = fit_task_costs(*data[0], *data[1:])
out = {"config": name, "costs": costs,
       "fitted_from": [{"D": r["D"], "N": r["N"], "partition": r["partition"]} for r in runs],
       "provenance": sys.argv[1],
       "units": "ms (W: per micro-batch) per stage-content term (attention / MLP half-block, LM head, "
                "embedding); isolated task times on one B200 (Trainer.measure_task_times)"}
dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2410_19367_b200",
                   "calibration", f"{name}.json")
with open(dst, "w") as f:
    json.dump(out, f, indent=1)
print(dst, json.dumps(costs))
