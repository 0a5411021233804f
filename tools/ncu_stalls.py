"""Warp-stall reason totals of an ncu --page source --csv dump (tools/ncu_stalls.py <src.csv>)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; tot = collections.Counter()
for r in rows:
    if len(r) > 3 and r[0] == 'Line No':
        hdr = r; cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]; continue
    if hdr is None or r[0] or len(r) < len(hdr) - 5: continue
    for i in cols:
        try: tot[hdr[i]] += float(r[i] or 0)
        except ValueError: pass
s = sum(tot.values()) or 1
print(' '.join(f"{k[6:]}={100*v/s:.1f}%" for k, v in tot.most_common(12)))
