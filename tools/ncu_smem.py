"""Per CUDA source line: shared-memory wavefronts (total / ideal / excessive), global L2 sectors,
warp instructions and stall samples, for every profiled instance of a kernel in an ncu report.

usage: ncu_smem.py REPORT KERNEL_REGEX [TOP]"""
import csv, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{pat}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
blocks, cur, fname, hdr, kname = [], None, None, None, None
for l in out:
    if l.startswith('"Kernel Name"') or l.startswith('"Function Name"'):
        kname = l
        continue
    if l.startswith('"File Path"'):
        fname = l.split(",", 1)[1].strip('"').split("/")[-1]
        continue
    if l.startswith('"Line No"'):
        hdr = next(csv.reader([l]))
        if cur is None or cur["k"] != kname or fname == "FIRST":
            pass
        cur = {"k": kname, "f": fname, "rows": []}
        blocks.append(cur)
        continue
    if not hdr or cur is None:
        continue
    r = next(csv.reader([l]))
    if not r or r[0] == "":
        continue
    try:
        f = lambda i: float(r[i] or 0)
        cur["rows"].append((r[0], r[1][:100].strip(), f(4), f(7), f(19), f(20), f(18), f(22), f(23)))
    except (ValueError, IndexError):
        pass
for b in blocks:
    rows = b["rows"]
    if not rows:
        continue
    tw = sum(x[4] for x in rows); ti = sum(x[3] for x in rows); ts = sum(x[2] for x in rows)
    if tw == 0 and ti == 0:
        continue
    print(f"=== {b['k'][:120]} | file {b['f']} | inst {ti:.0f} samples {ts:.0f} smem wavefronts {tw:.0f} ideal {sum(x[5] for x in rows):.0f}")
    for x in sorted(rows, key=lambda x: -x[4])[:top]:
        print(f"  L{x[0]:>5} wf {x[4]/max(tw,1)*100:5.1f}% (x{x[4]/max(x[5],1):4.1f} ideal) inst {x[3]/max(ti,1)*100:5.1f}% stall {x[2]/max(ts,1)*100:5.1f}% glob {x[7]:.0f}/{x[8]:.0f} | {x[1]}")
