"""Summarise an ncu --set full report of lz_step_kernel: key raw metrics + SASS opcode mix + top stalls."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum', 'launch__grid_size',
        'lts__t_sector_hit_rate.pct', 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'smsp__cycles_active.avg', 'sm__cycles_elapsed.avg']
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
raw_hdr, raw_row = rows[0], rows[2]
for r in rows[2:]:
    print(r[hdr.index('Kernel Name')][:80])
    for w in WANT:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w:62s} {r[i]:>16s} {units[i]}")
src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source=sass'], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
blocks, cur, hdr = [], None, None
for r in rows:
    if r and r[0] == 'Kernel Name':
        cur = []
        blocks.append(cur)
        continue
    if r and r[0] == 'Address':
        hdr = r
        continue
    if cur is not None and len(r) > 5:
        cur.append(r)
data = blocks[0]
si = hdr.index('Warp Stall Sampling (All Samples)')
ii = hdr.index('Instructions Executed')
f = lambda x: float(x) if x not in ('', '-') else 0.0
ts = sum(f(r[si]) for r in data)
ti = sum(f(r[ii]) for r in data)
print(f"SASS lines {len(data)}  stall samples {ts:.0f}  warp instructions {ti:.4g}")
byop, bys = collections.Counter(), collections.Counter()
for r in data:
    t = r[1].split()
    op = t[1] if t[0].startswith('@') else t[0]
    byop[op] += f(r[ii])
    bys[op] += f(r[si])
for op, c in byop.most_common(16):
    print(f"  {op:22s} instr {100 * c / ti:5.1f}%  stall-samples {100 * bys[op] / ts:5.1f}%")
stall_cols = [h for h in hdr if h.startswith('stall_') or 'Stall Reasons' in h]

# stall reasons (pc sampling), largest first
vals = []
for i, n in enumerate(raw_hdr):
    if 'pcsamp_warps_issue_stalled' in n and not n.endswith('not_issued'):
        try:
            vals.append((float(raw_row[i].replace(',', '')), n))
        except (ValueError, IndexError):
            pass
tot = sum(v for v, _ in vals) or 1.0
print("stall reasons (pc samples):")
for v, n in sorted(vals, reverse=True)[:12]:
    print(f"  {n.replace('smsp__pcsamp_warps_issue_stalled_', ''):32s} {100 * v / tot:5.1f}%")
