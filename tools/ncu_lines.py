"""Per-source-line instruction / stall-sample totals of one kernel from an ncu
report (--page source --print-source cuda,sass CSV).  Usage:
    ncu -i REP --page source --csv -k regex:NAME --print-source cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
ie = h.index("Instructions Executed")
ws = h.index("Warp Stall Sampling (All Samples)")
acc = {}
for r in rows[hi + 1:]:
    # line-level aggregate rows carry the line number; SASS rows have it empty
    if len(r) <= ie or not r[0].isdigit():
        continue
    cur = (int(r[0]), r[1][:90])
    try:
        n = float(r[ie] or 0)
        s = float(r[ws] or 0)
    except ValueError:
        continue
    a = acc.setdefault(cur, [0.0, 0.0])
    a[0] += n
    a[1] += s
tot_i = sum(v[0] for v in acc.values()) or 1
tot_s = sum(v[1] for v in acc.values()) or 1
print(f"total instr {tot_i:.0f}  samples {tot_s:.0f}")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]:5d} {100*v[0]/tot_i:5.1f}% inst {100*v[1]/tot_s:5.1f}% samp  {k[1]}")
