"""Key per-launch metrics of an ncu --set full report (one row per launch).

usage: ncu_key.py REPORT [substring ...]   (extra metric-name substrings to print)"""
import csv, subprocess, sys
rep = sys.argv[1]
extra = sys.argv[2:]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h = rr[0]
want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_lsu.sum", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__cycles_elapsed.max"]
cols = [c for c in h if c in want or any(e in c for e in extra)]
ki = h.index("Kernel Name")
for r in rr[2:]:
    if len(r) < len(h):
        continue
    print("==", r[ki].split("(")[0][:60])
    for c in cols:
        print(f"   {c:75s} {r[h.index(c)]}")
    if "stall" in extra or True:
        st = [(c, r[h.index(c)]) for c in h if "smsp__average_warps_issue_stalled" in c and "per_issue_active" in c and "not_issued" not in c]
        st = sorted(st, key=lambda x: -float(x[1].replace(",", "") or 0))[:6]
        for c, v in st:
            print(f"   stall {c.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):40s} {v}")
