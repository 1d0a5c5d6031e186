"""Per-source-line warp-stall samples of each kernel in an ncu --set full --import-source report."""
import csv
import subprocess
import sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source=cuda,sass'], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
blocks, cur = [], None
for r in rows:
    if r and r[0] == 'Function Name':
        cur = {'name': r[1], 'rows': []}
        blocks.append(cur)
    elif r and r[0] == 'Line No':
        cur['hdr'] = r
    elif cur is not None and 'hdr' in cur and len(r) > 4 and r[2] == '-':
        cur['rows'].append(r)
for b in blocks:
    k = b['hdr'].index('Warp Stall Sampling (All Samples)')
    data = [(float(r[k]), r[0], r[1][:100]) for r in b['rows'] if r[k] not in ('', '0')]
    tot = sum(d[0] for d in data) or 1.0
    print(f"== {b['name'][:90]}  ({int(tot)} samples)")
    for d in sorted(data, reverse=True)[:top]:
        print(f"  {100 * d[0] / tot:5.1f}% L{d[1]:>4} {d[2]}")
