"""Summarize an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes])."""
import csv, collections, sys
path = sys.argv[1]
skip_torch = True
rows = list(csv.reader(open(path)))
for i, r in enumerate(rows):
    if 'Kernel Name' in r:
        hdr = r; start = i + 1; break
ki, vi, mi, ii = (hdr.index(k) for k in ('Kernel Name', 'Metric Value', 'Metric Name', 'ID'))
gi = hdr.index('Grid Size')
per = collections.OrderedDict()
for r in rows[start:]:
    if len(r) <= vi: continue
    d = per.setdefault(r[ii], {'name': r[ki].replace('void ', '').replace('acct::', '').replace('<unnamed>::', '').split('(')[0], 'grid': r[gi]})
    d[r[mi]] = float(r[vi].replace(',', ''))
L = [d for d in per.values() if not (skip_torch and d['name'].startswith('at::'))]
n = int(sys.argv[2]) if len(sys.argv) > 2 else len(L)
L = L[-n:]
tot = sum(d.get('gpu__time_duration.sum', 0) for d in L)
for d in L:
    t = d.get('gpu__time_duration.sum', 0)
    rb = d.get('dram__bytes_read.sum', 0); wb = d.get('dram__bytes_write.sum', 0)
    print(f"{t/1000:8.2f} us {100*t/tot:5.1f}%  R{rb/1e6:7.2f}MB W{wb/1e6:6.2f}MB  {d['grid']:>14}  {d['name']}")
print(f"total {tot/1000:.1f} us over {len(L)} launches")
