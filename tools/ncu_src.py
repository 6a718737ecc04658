"""Hottest CUDA source lines (warp-stall samples, instructions) of a kernel in an ncu report.

Uses the cuda,sass source view (needs -lineinfo + --import-source on)."""
import csv, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{pat}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
res, fname, hdr, seen_fn = [], None, None, set()
for l in out:
    if l.startswith('"File Path"'):
        fname = l.split(",", 1)[1].strip('"').split("/")[-1]
        continue
    if l.startswith('"Function Name"'):
        seen_fn.add(l)
        if len(seen_fn) > 1:  # first matching kernel only
            break
        continue
    if l.startswith('"Line No"'):
        hdr = next(csv.reader([l]))
        continue
    if not hdr:
        continue
    r = next(csv.reader([l]))
    if not r or r[0] == "":
        continue
    try:
        txt = r[1]
        res.append((int(r[4] or 0), int(float(r[7] or 0)), fname, r[0], txt[:110]))
    except (ValueError, IndexError):
        pass
tot = sum(r[0] for r in res) or 1
toti = sum(r[1] for r in res) or 1
print(f"total samples {tot}  warp-inst {toti}")
for r in sorted(res, key=lambda r: -r[0])[:top]:
    print(f"{100*r[0]/tot:5.1f}% stall {100*r[1]/toti:5.1f}% inst  {r[2]}:{r[3]}  {r[4].strip()}")
