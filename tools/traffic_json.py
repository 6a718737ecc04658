"""profiles/<tag>_traffic_c<cfg>.json from an ncu launch list (gpu__time_duration,
dram__bytes_read/write per launch) of ONE sort: DRAM bytes per kernel family
per sort, which bench.py reports as roofline.traffic for the dominant phase.

    python tools/traffic_json.py gpurun_out/r02b_launches_c4.csv 4 100000000 profiles/r02b_traffic_c4.json
"""
import collections
import csv
import json
import sys

src, cfg, n, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
rows = list(csv.reader(open(src)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    per.setdefault((int(r[ii]), r[ki].split("(")[0].replace("void ", "").split("<")[0]), {})[r[mi]] = float(
        r[vi].replace(",", ""))
fam = collections.defaultdict(float)
tim = collections.defaultdict(float)
for (_, name), m in per.items():
    fam[name] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    tim[name] += m.get("gpu__time_duration.sum", 0) / 1e3
alias = {"k_team": "k_finish", "k_refine": "k_finish", "k_level1_map": "k_moments", "k_seg_moments": "k_recursion_stats"}
bps = collections.defaultdict(float)
for k, v in fam.items():
    bps[alias.get(k, k)] += v
json.dump({"source": src, "config": cfg, "n": n, "bytes_per_step": dict(bps),
           "ncu_us_per_step": dict(tim)}, open(out, "w"), indent=1)
print(json.dumps(dict(bps), indent=1))
