"""Per CUDA source line of sort_kernels.cuh/common.cuh: warp instructions and stall samples (top by instructions),
first profiled instance of the kernel.  usage: ncu_lines.py REPORT KERNEL_REGEX [TOP]"""
import csv, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{pat}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows, fname, hdr, seen = [], None, None, []
for l in out:
    if l.startswith('"Kernel Name"') or l.startswith('"Function Name"'):
        if l not in seen:
            seen.append(l)
        if len(seen) > 1:
            break
        continue
    if l.startswith('"File Path"'):
        fname = l.split(",", 1)[1].strip('"').split("/")[-1]
        continue
    if l.startswith('"Line No"'):
        hdr = True
        continue
    if not hdr:
        continue
    r = next(csv.reader([l]))
    if not r or r[0] == "":
        continue
    try:
        rows.append((fname, r[0], r[1][:95].strip(), float(r[4] or 0), float(r[7] or 0)))
    except (ValueError, IndexError):
        pass
ti = sum(x[4] for x in rows) or 1
ts = sum(x[3] for x in rows) or 1
print(seen[0][:140], "inst", ti, "samples", ts)
for x in sorted(rows, key=lambda x: -x[4])[:top]:
    print(f"  {x[0][:18]:18s} L{x[1]:>5} inst {x[4]/ti*100:5.1f}% stall {x[3]/ts*100:5.1f}% | {x[2]}")
