"""Select the columns profiles/*_ncu_full_summary.csv holds from an `ncu -i X.ncu-rep --page raw --csv` dump.
usage: ncu -i prof.ncu-rep --page raw --csv > raw.csv; python tools/ncu_summary.py raw.csv > summary.csv"""
import csv, re, sys
COLS = """launch__grid_size launch__block_size launch__registers_per_thread gpu__time_duration.sum dram__bytes_read.sum
dram__bytes_write.sum gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed lts__t_sectors.sum lts__t_sector_hit_rate.pct
lts__throughput.avg.pct_of_peak_sustained_elapsed l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed
sm__throughput.avg.pct_of_peak_sustained_elapsed sm__warps_active.avg.pct_of_peak_sustained_active
smsp__issue_active.avg.pct_of_peak_sustained_active sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active
sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed smsp__inst_executed.sum
smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio
smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio
smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio
smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio
smsp__average_warps_issue_stalled_wait_per_issue_active.ratio""".split()
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
names, units, data = rows[hdr], rows[hdr + 1], rows[hdr + 2:]
ki = names.index("Kernel Name")
idx = [names.index(c) if c in names else -1 for c in COLS]
out = csv.writer(sys.stdout)
out.writerow(["Kernel Name"] + COLS)
out.writerow([""] + [units[i] if i >= 0 else "" for i in idx])
seen = set()
for r in data:
    name = re.sub(r"\(.*", "", r[ki]).replace("gapa_b200::", "").replace("void ", "")
    if name in seen:  # first launch of each kernel
        continue
    seen.add(name)
    out.writerow([name] + [r[i] if i >= 0 else "" for i in idx])
