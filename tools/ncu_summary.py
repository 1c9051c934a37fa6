"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
rows = list(csv.reader(open(path)))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
unit_i = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    u = r[unit_i] if unit_i is not None else "ns"
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(u, 1e-3)
    name = r[ki]
    short = name.split("(")[0][:90]
    tot[short] += v * scale
    cnt[short] += 1
T = sum(tot.values())
print(f"total kernel time {T/1e3:.2f} ms over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:40]:
    print(f"{v/1e3:9.3f} ms {100*v/T:5.1f}%  n={cnt[k]:6d}  avg {v/cnt[k]:8.1f} us  {k}")
