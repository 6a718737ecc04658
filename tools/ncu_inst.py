"""Top SASS lines of a kernel by executed warp instructions (the profiled
instance of that kernel with the most instructions)."""
import csv, io, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{pat}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
blocks, cur = [], None
for l in lines:
    if l.startswith('"Kernel Name"'):
        cur = []
        blocks.append(cur)
    elif cur is not None:
        cur.append(l)
best, best_tot = None, -1
for b in blocks:
    rows = list(csv.reader(io.StringIO("\n".join(b))))
    h = rows[0]
    ii = h.index("Instructions Executed")
    tot = sum(float(r[ii] or 0) for r in rows[1:] if len(r) > ii)
    if tot > best_tot:
        best, best_tot = rows, tot
h = best[0]
ii, si = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
stot = sum(float(r[si] or 0) for r in best[1:])
print("total inst", best_tot, "samples", stot)
mode = sys.argv[4] if len(sys.argv) > 4 else "inst"
key = ii if mode == "inst" else si
for r in sorted(best[1:], key=lambda r: -float(r[key] or 0))[:top]:
    print(f"{float(r[ii])/best_tot*100:5.1f}% inst {float(r[si] or 0)/max(stot,1)*100:5.1f}% stall  {r[1].strip()[:100]}")
