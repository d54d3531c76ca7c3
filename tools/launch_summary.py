"""Summarise an ncu launch list (gpu__time_duration.sum CSV) per kernel:
count, mean duration and share of the summed kernel time.
Usage: launch_summary.py LAUNCHES.csv "header comment" > profiles/rNN_launches_summary.txt"""
import csv, sys
from collections import OrderedDict
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
kn, mv = hdr.index("Kernel Name"), hdr.index("Metric Value")
acc = OrderedDict()
for r in rows[1:]:
    name = r[kn].replace("void ", "").split("(")[0].replace("stereo::", "")
    acc.setdefault(name, []).append(float(r[mv]))
tot = sum(sum(v) for v in acc.values())
print(f"# {sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]}")
print("# kernel  n  avg_ns  share_of_step")
for k, v in acc.items():
    print(f"{k:28s} {len(v):4d} {sum(v) / len(v):10.0f} {100 * sum(v) / tot:5.1f}%")
