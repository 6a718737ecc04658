"""Top SASS lines of a kernel by executed warp instructions, with CUDA source line when available."""
import csv, io, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
mode = sys.argv[4] if len(sys.argv) > 4 else "sass"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{pat}", "--print-source", mode],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"') or l.startswith('"Line"') or l.startswith('"#"'))
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"Kernel Name"')), len(lines))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:end]))))
h = rows[0]
ii = h.index("Instructions Executed")
si = h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[ii] or 0) for r in rows[1:])
stot = sum(float(r[si] or 0) for r in rows[1:])
print("total inst", tot, "samples", stot)
for r in sorted(rows[1:], key=lambda r: -float(r[ii] or 0))[:top]:
    print(f"{float(r[ii])/tot*100:5.1f}% inst {float(r[si] or 0)/max(stot,1)*100:5.1f}% stall  {r[0][:6]} {r[1].strip()[:100]}")
