"""Summarise an ncu --set full report (raw CSV page) per kernel."""
import csv, sys
path = sys.argv[1]
rows = list(csv.reader(open(path)))
hdr, units = rows[0], rows[1]
want = [
    ("gpu__time_duration.sum", "dur"), ("sm__cycles_elapsed.avg.per_second", "clk"),
    ("smsp__inst_executed.sum", "inst"), ("sm__inst_executed.avg.per_cycle_active", "ipc"),
    ("dram__bytes_read.sum", "dramR"), ("dram__bytes_write.sum", "dramW"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("lts__t_bytes.sum", "L2bytes"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smemWF"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bankConf"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "shpipe%"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "st_bar"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "st_lsb"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "st_ssb"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "st_mio"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "st_wait"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "st_math"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "st_lg"),
]
idx = {h: i for i, h in enumerate(hdr)}
for r in rows[2:]:
    name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "").replace("stereo::", "")[:26]
    out = [name]
    for m, short in want:
        if m in idx:
            v = r[idx[m]]
            out.append(f"{short}={v}{units[idx[m]] if units[idx[m]] not in ('', 'inst') else ''}")
    print("  ".join(out))
