"""Summarise a multi-metric ncu launch list (gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum,
lts__t_bytes.sum; --csv): per kernel name the device time, DRAM and L2 bytes per launch and the achieved L2 / DRAM
bandwidth. Usage: python scripts/launch_summary_mem.py launches.csv [note]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == 'ID'][0]
hdr = rows[i]
ki, vi, ui, mi, ii = (hdr.index(c) for c in ('Kernel Name', 'Metric Value', 'Metric Unit', 'Metric Name', 'ID'))
tscale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}
bscale = {'byte': 1.0, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'KB': 1e3, 'MB': 1e6, 'GB': 1e9}
per = collections.defaultdict(dict)
names = {}
for r in rows[i + 1:]:
    if len(r) <= vi:
        continue
    name = re.sub(r'^void\s+', '', r[ki])
    name = re.sub(r'\(.*$', '', name).replace('<unnamed>::', '').replace('(anonymous namespace)::', '')
    names[r[ii]] = name
    v = float(r[vi].replace(',', ''))
    u = r[ui]
    per[r[ii]][r[mi]] = v * (tscale[u] if r[mi] == 'gpu__time_duration.sum' else bscale.get(u, 1.0))
agg = collections.defaultdict(lambda: collections.Counter())
for lid, m in per.items():
    a = agg[names[lid]]
    a['n'] += 1
    a['us'] += m.get('gpu__time_duration.sum', 0.0)
    a['dram'] += m.get('dram__bytes_read.sum', 0.0) + m.get('dram__bytes_write.sum', 0.0)
    a['l2'] += m.get('lts__t_bytes.sum', 0.0)
T = sum(a['us'] for a in agg.values())
print(f"{sum(a['n'] for a in agg.values())} launches, {T / 1e3:.3f} ms device time (serialised under ncu) "
      f"{sys.argv[2] if len(sys.argv) > 2 else ''}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]['us']):
    us = a['us']
    print(f"  {k:42s} n={a['n']:4d} {us / 1e3:8.3f} ms {100 * us / T:5.1f}%  per launch {us / a['n']:8.1f} us, "
          f"DRAM {a['dram'] / a['n'] / 1e6:8.2f} MB, L2 {a['l2'] / a['n'] / 1e6:8.2f} MB -> "
          f"DRAM {a['dram'] / us / 1e3:6.0f} GB/s, L2 {a['l2'] / us / 1e3:6.0f} GB/s")
