"""Write profiles/<tag>_summary.md from a gpu_profile_round.sh capture."""
import collections, csv, json, subprocess, sys, os
tag = sys.argv[1]
d = "gpurun_out"
out = []
bench = json.loads(open(f"{d}/{tag}_bench.json").read().strip().splitlines()[-1])
out.append(f"# Profile summary {tag}\n")
out.append("GPU: " + " / ".join(open(f"{d}/{tag}_gpu.txt").read().strip().splitlines()[1:]) + "\n")
out.append("## bench.py line (default workload)\n\n```json\n" + json.dumps(bench, indent=1) + "\n```\n")
rows = list(csv.reader(open(f"{d}/{tag}_launches.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    per.setdefault((int(r[ii]), r[ki].split("(")[0]), {})[r[mi]] = float(r[vi].replace(",", ""))
items = list(per.items())
# last full sort: from the last k_init_level1 on
inits = [i for i, ((_, n), _) in enumerate(items) if "k_init_level1" in n or "k_level1_map" in n]
start, stop = (inits[-2], inits[-1]) if len(inits) >= 2 else (inits[-1], len(items))
step = [(k, m) for k, m in items[start:stop] if "at::" not in k[1] and "k_check" not in k[1]]
tot = sum(m.get("gpu__time_duration.sum", 0) for _, m in step)
out.append("## ncu launch list, one sort (cold-cache, serialised; compare shares)\n")
out.append("| # | kernel | time us | share | DRAM read MB | DRAM write MB | GB/s |\n|---|---|---|---|---|---|---|")
for (i, name), m in step:
    t = m.get("gpu__time_duration.sum", 0)
    rd, wr = m.get("dram__bytes_read.sum", 0), m.get("dram__bytes_write.sum", 0)
    out.append(f"| {i} | {name} | {t/1e3:.1f} | {100*t/tot:.1f}% | {rd/1e6:.1f} | {wr/1e6:.1f} | {(rd+wr)/max(t,1):.0f} |")
out.append(f"\nSum of kernel time for one sort: {tot/1e3:.1f} us\n")
raw = subprocess.run(["ncu", "-i", f"{d}/{tag}_full.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
if rr:
    h = rr[0]
    out.append("## ncu --set full (hot kernels)\n")
    out.append("| kernel | us | DRAM rd MB | DRAM wr MB | DRAM % peak | issue active % | warps active % | top stalls |\n|---|---|---|---|---|---|---|---|")
    traffic = {}
    for r in rr[2:]:
        dd = {h[i]: r[i] for i in range(len(h))}
        kname = dd.get("Kernel Name", "").split("(")[0].replace("void ", "").replace("zsb::", "").split("<")[0]
        mb = float(dd.get("dram__bytes_read.sum", "0") or 0) + float(dd.get("dram__bytes_write.sum", "0") or 0)
        traffic.setdefault(kname, []).append(mb * 1e6)
        st = [(k, float(dd[k].replace(",", ""))) for k in dd if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and dd[k] not in ("", "n/a")]
        stt = sum(v for _, v in st) or 1
        top = ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_','')} {100*v/stt:.0f}%" for k, v in sorted(st, key=lambda x: -x[1])[:3])
        f = lambda k: dd.get(k, "")
        out.append(f"| {f('Kernel Name').split('(')[0]} | {float(f('gpu__time_duration.sum')):.1f} | {float(f('dram__bytes_read.sum')):.1f} | {float(f('dram__bytes_write.sum')):.1f} | "
                   f"{f('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')[:5]} | {f('smsp__issue_active.avg.pct_of_peak_sustained_active')[:5]} | "
                   f"{f('sm__warps_active.avg.pct_of_peak_sustained_active')[:5]} | {top} |")
os.makedirs("profiles", exist_ok=True)
open(f"profiles/{tag}_summary.md", "w").write("\n".join(out) + "\n")
if rr:  # DRAM bytes (read + write) per launch of each captured kernel, for bench.py's roofline.traffic
    json.dump({"source": f"profiles/{tag}_summary.md (ncu --set full)", "bytes_per_launch": traffic},
              open(f"profiles/{tag}_traffic.json", "w"), indent=1)
import shutil
for suffix in ("launches.csv", "bench.json"):
    shutil.copy(f"{d}/{tag}_{suffix}", f"profiles/{tag}_{suffix}")
print("\n".join(out))
