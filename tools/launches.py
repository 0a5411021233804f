"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: last step's kernels."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; out = []
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            out.append((d['Kernel Name'], float(d['Metric Value']) * (1e-3 if d['Metric Unit'] == 'ns' else 1.0)))
first = sys.argv[2] if len(sys.argv) > 2 else 'k_fiber_bound'
idx = [i for i, o in enumerate(out) if first in o[0]]
last = out[idx[-1]:] if idx else out
agg = collections.OrderedDict()
for name, us in last:
    short = name.split('(')[0].replace('void ', '')[:60]
    agg.setdefault(short, [0, 0.0]); agg[short][0] += 1; agg[short][1] += us
tot = sum(v[1] for v in agg.values())
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{us/1e3:9.3f} ms {100*us/tot:5.1f}%  x{n:3d}  {k}")
print(f"{tot/1e3:9.3f} ms total, {sum(v[0] for v in agg.values())} launches")
