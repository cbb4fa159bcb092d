"""Summarise an ncu report: SOL, occupancy, dram bytes, top stalls / opcodes."""
import collections, csv, subprocess, sys

def page(rep, name):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))

rep = sys.argv[1]
r = page(rep, "details")
h = r[0]
want = {'Duration', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Executed Ipc Active', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Issue Slots Busy', 'No Eligible', 'Warp Cycles Per Issued Instruction', 'Dynamic Shared Memory Per Block',
        'Grid Size', 'Block Size', 'Waves Per SM'}
for row in r[1:]:
    d = dict(zip(h, row))
    if d.get('Metric Name') in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']:>12s} {d.get('Metric Unit','')}")
raw = page(rep, "raw")
if len(raw) > 2:
    hh = raw[0]
    vals = raw[2] if len(raw) > 2 else raw[1]
    d = dict(zip(hh, vals))
    for k in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active'):
        if k in d:
            print(f"{k:40s} {d[k]:>12s} {raw[1][hh.index(k)]}")
src = page(rep, "source")
if len(src) > 2:
    hh = src[1]
    rows = [dict(zip(hh, x)) for x in src[2:]]
    agg = collections.Counter(); stall = collections.Counter(); tot = 0
    for d in rows:
        op = d.get('Source', '').strip().split()
        if not op: continue
        o = op[1] if op[0].startswith('@') else op[0]
        o = o.split('.')[0]
        n = float(d.get('Instructions Executed') or 0); agg[o] += n; tot += n
        stall[o] += float(d.get('Warp Stall Sampling (All Samples)') or 0)
    print('warp instructions', tot)
    for o, n in agg.most_common(12):
        print(f"  {o:10s} {n / max(tot, 1) * 100:5.1f}%  stall-samples {stall[o]:.0f}")
    rows.sort(key=lambda d: -float(d.get('Warp Stall Sampling (All Samples)') or 0))
    print('top stall instructions:')
    for d in rows[:10]:
        print('  ', d.get('Warp Stall Sampling (All Samples)'), d.get('Address', '')[-5:], d.get('Source', '').strip()[:90])
