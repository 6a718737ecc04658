"""Sum warp-instructions and stall samples of a kernel by source-line ranges of one file.

usage: ncu_ranges.py REPORT KERNEL_REGEX FILE name:lo-hi [name:lo-hi ...]"""
import csv, subprocess, sys
rep, pat, fname = sys.argv[1], sys.argv[2], sys.argv[3]
ranges = [(a.split(":")[0], *map(int, a.split(":")[1].split("-"))) for a in sys.argv[4:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{pat}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
cur, seen, acc, other = None, set(), {r[0]: [0, 0] for r in ranges}, [0, 0]
hdr = None
for l in out:
    if l.startswith('"File Path"'):
        cur = l.split(",", 1)[1].strip('"').split("/")[-1]
        continue
    if l.startswith('"Function Name"'):
        seen.add(l)
        if len(seen) > 1:
            break
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
        st, ins, ln = int(r[4] or 0), int(float(r[7] or 0)), int(r[0])
    except (ValueError, IndexError):
        continue
    hit = False
    if cur == fname:
        for name, lo, hi in ranges:
            if lo <= ln <= hi:
                acc[name][0] += ins
                acc[name][1] += st
                hit = True
                break
    if not hit:
        other[0] += ins
        other[1] += st
ti = sum(v[0] for v in acc.values()) + other[0]
ts = sum(v[1] for v in acc.values()) + other[1]
for name, (i, s) in list(acc.items()) + [("other/inlined", tuple(other))]:
    print(f"{name:16s} inst {100*i/ti:5.1f}%  stall {100*s/ts:5.1f}%")
print("total warp-inst", ti)
