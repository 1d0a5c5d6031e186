"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): time share per kernel."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == 'ID'][0]
hdr = rows[i]
ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
mi = hdr.index('Metric Name')
scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[i + 1:]:
    if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':  # other metrics of the same capture are ignored
        continue
    name = re.sub(r'^void\s+', '', r[ki])
    name = re.sub(r'\(.*$', '', name).replace('<unnamed>::', '').replace('(anonymous namespace)::', '')
    tot[name] += float(r[vi].replace(',', '')) * scale[r[ui]]
    cnt[name] += 1
T = sum(tot.values())
print(f"{sum(cnt.values())} launches, {T / 1e3:.3f} ms total device time (cold-cache, serialised under ncu)")
for k, v in tot.most_common():
    print(f"  {k:55s} n={cnt[k]:4d}  {v / 1e3:9.3f} ms  {100 * v / T:5.1f}%  mean {v / cnt[k]:10.1f} us")
