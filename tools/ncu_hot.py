"""Print the hottest SASS lines (by warp-stall samples) of a kernel in an ncu report."""
import csv, io, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{pat}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"Kernel Name"')), len(lines))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:end]))))
h = rows[0]
si = h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[si] or 0) for r in rows[1:])
best = sorted(rows[1:], key=lambda r: -int(r[si] or 0))[:top]
print("total samples", tot)
for r in best:
    print(f"{int(r[si])/max(tot,1)*100:5.1f}%  {r[1].strip()[:90]}")
