"""Per-kernel launch counts and last durations (ms) from an ncu --csv launch list.
usage: python tools/launch_summary.py LAUNCHES.csv [substring ...]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
keys = sys.argv[2:]
h, d = None, collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h and len(r) == len(h):
        d[r[h.index("Kernel Name")].split("(")[0][-48:]].append(float(r[h.index("Metric Value")].replace(",", "")))
for k, v in d.items():
    if not keys or any(s in k for s in keys):
        print(f"{k:50s} {len(v):4d}  " + " ".join(f"{x / 1e6:.3f}" for x in v[-4:]))
