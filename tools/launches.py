"""Summarise an ncu --csv launch list: per-kernel time and DRAM bytes (last N launches)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    per.setdefault((int(r[ii]), r[ki].split('(')[0][:48]), {})[r[mi]] = float(r[vi].replace(',', ''))
last = int(sys.argv[2]) if len(sys.argv) > 2 else 12
tot = 0
for (i, name), m in list(per.items())[-last:]:
    t = m.get('gpu__time_duration.sum', 0)
    tot += t
    rd, wr = m.get('dram__bytes_read.sum', 0), m.get('dram__bytes_write.sum', 0)
    print(f"{i:4d} {name:48s} {t/1e3:9.1f} us  rd {rd/1e6:8.1f} MB  wr {wr/1e6:8.1f} MB  {(rd+wr)/max(t,1):7.1f} GB/s")
print(f"sum {tot/1e3:.1f} us")
