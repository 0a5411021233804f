"""From an ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv launch
list of `bench.py --steps 1 --warmup 1`: per-kernel time and DRAM bytes of the LAST step (from the
last k_fiber_bound / first kernel given), as JSON (used for bench.py's roofline.traffic)."""
import csv, sys, json, collections
rows = list(csv.reader(open(sys.argv[1])))
first = sys.argv[2] if len(sys.argv) > 2 else 'k_fiber_bound'
hdr = None
launch = collections.OrderedDict()
for r in rows:
    if r and r[0] == 'ID':
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = (d['ID'], d['Kernel Name'])
        e = launch.setdefault(k, {})
        v = float(d['Metric Value'].replace(',', '') or 0)
        u = d['Metric Unit']
        if d['Metric Name'] == 'gpu__time_duration.sum':
            e['ms'] = v * {'ns': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'nsecond': 1e-6, 'ms': 1.0, 'msecond': 1.0}.get(u, 1e-6)
        else:
            e[d['Metric Name']] = v * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'KB': 1e3, 'MB': 1e6, 'GB': 1e9}.get(u, 1)
items = list(launch.items())
idx = [i for i, ((_, n), _) in enumerate(items) if first in n]
items = items[idx[-1]:] if idx else items
agg = collections.OrderedDict()
for (_, name), e in items:
    short = name.split('(')[0].replace('void ', '').split('<')[0].replace('vox::', '')
    a = agg.setdefault(short, {'launches': 0, 'ms': 0.0, 'dram_bytes': 0.0})
    a['launches'] += 1
    a['ms'] += e.get('ms', 0.0)
    a['dram_bytes'] += e.get('dram__bytes_read.sum', 0.0) + e.get('dram__bytes_write.sum', 0.0)
json.dump(agg, sys.stdout, indent=1)
