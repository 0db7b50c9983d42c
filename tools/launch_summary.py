"""Summarise an `ncu --csv` launch list: one generation's kernels in order + totals per kernel."""
import collections, csv, re, sys
path = sys.argv[1]
anchor = sys.argv[2] if len(sys.argv) > 2 else "k_pc_reset"
hdr = None; rows = []
for line in csv.reader(open(path)):
    if 'Kernel Name' in line: hdr = line; continue
    if hdr and len(line) == len(hdr): rows.append(line)
ki, mi, vi, ui, ii = (hdr.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
per = collections.OrderedDict()
for r in rows:
    d = per.setdefault(r[ii], {'name': re.sub(r'\(.*', '', r[ki]).replace('gapa_b200::', '').replace('void ', '')})
    v = float(r[vi].replace(',', '')); u = r[ui]
    if r[mi].startswith('gpu__time'):
        v = v / 1e3 if u.startswith('ns') else (v * 1e3 if u.startswith('ms') else v)
    elif 'bytes' in r[mi]:
        v = v * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}[u] / 1e6
    d[r[mi]] = v
seq = list(per.values())
idx = [i for i, d in enumerate(seq) if d['name'] == anchor]
a, b = (idx[1], idx[2]) if len(idx) > 2 else (0, len(seq))
tot = 0
print(f"one step ({anchor} .. next {anchor}):")
for d in seq[a:b]:
    t = d['gpu__time_duration.sum']; tot += t
    print(f"  {d['name']:30s} {t:9.1f} us  dram R {d.get('dram__bytes_read.sum', 0):8.1f} MB  W {d.get('dram__bytes_write.sum', 0):8.1f} MB  L2 {d.get('lts__t_sectors.sum', 0) / 1e6:8.1f} Msect")
print(f"  {'sum':30s} {tot:9.1f} us")
for d in seq[a:b]:
    d['share'] = d['gpu__time_duration.sum'] / tot
