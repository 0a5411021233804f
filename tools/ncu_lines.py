"""Aggregate an ncu --page source --csv --print-source cuda,sass dump per CUDA source line."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = {}
hdr = None
cur = None
for r in rows:
    if len(r) > 3 and r[0] == 'Line No':
        hdr = r; samp = hdr.index('Warp Stall Sampling (All Samples)'); ie = hdr.index('Instructions Executed'); continue
    if hdr is None or len(r) < len(hdr) - 5:
        continue
    if r[0]:
        cur = (r[0], r[1]); out.setdefault(cur, [0.0, 0.0])
        continue
    if cur:
        try:
            out[cur][0] += float(r[samp] or 0); out[cur][1] += float(r[ie] or 0)
        except ValueError:
            pass
tot = sum(v[0] for v in out.values()) or 1
for (ln, src), v in sorted(out.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{ln:>5} {100*v[0]/tot:5.1f}% inst={v[1]:10.3g}  {src.strip()[:95]}")
