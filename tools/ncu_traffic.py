"""Write profiles/ncu_traffic.json (DRAM bytes per launch, from one ncu --set full
capture) for bench.py's roofline.traffic field.  Usage: ncu_traffic.py RAW.csv TAG"""
import csv, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (the source digest bench.py checks before using this file)
rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = {"source": f"ncu --set full --clock-control none, report {os.path.basename(sys.argv[1])} ({sys.argv[2]})",
       "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch; writes still dirty in L2 at kernel end are not counted",
       "frames_per_launch": int(os.environ.get("QT_BATCH", "1")),
       "source_sha": bench._source_sha()}
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
    # pipe utilisation (the bound of the aggregation kernels is issue / shared
    # memory, not HBM): percentages of peak over active cycles
    def g(m):
        try:
            return float(r[hdr.index(m)])
        except (ValueError, IndexError):
            return None
    cyc = g("sm__cycles_elapsed.avg") or None
    wf = g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
    nsm = g("device__attribute_multiprocessor_count") or 148.0
    out.setdefault("pipes", {})[key] = {
        "issue_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "alu_pct": g("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "lsu_pct": g("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
        "smem_wavefronts_per_sm_cycle": (wf / nsm / cyc) if (wf and cyc) else None,
        "bank_conflict_wavefronts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "duration_ns": (g("gpu__time_duration.sum") or 0) * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(
            units[hdr.index("gpu__time_duration.sum")], 1),
    }
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
