"""Write profiles/ncu_traffic.json (DRAM bytes per launch, from one ncu --set full
capture) for bench.py's roofline.traffic field.  Usage: ncu_traffic.py RAW.csv TAG"""
import csv, json, os, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = {"source": f"ncu --set full --clock-control none, report {os.path.basename(sys.argv[1])} ({sys.argv[2]})",
       "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch; writes still dirty in L2 at kernel end are not counted"}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    key = next((k for k in ("sd", "prep", "xpass", "ypass", "post") if name.replace("void ", "").replace("stereo::", "").startswith(k)), None)
    if not key:
        continue
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(m)
        tot += float(r[i]) * scale[units[i]]
    out[key] = int(tot)
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
