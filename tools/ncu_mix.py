"""Per-line and per-opcode instruction mix of an ncu --page source --csv --print-source cuda,sass dump:
instructions executed, shared-memory wavefronts and warp-stall samples (tools/ncu_mix.py <src.csv> [n])."""
import csv, sys, re, collections
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None; cur = None
lines = collections.defaultdict(lambda: [0.0, 0.0, 0.0, ''])
ops = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for r in rows:
    if len(r) > 3 and r[0] == 'Line No':
        hdr = r; ie = hdr.index('Instructions Executed'); samp = hdr.index('Warp Stall Sampling (All Samples)')
        wf = hdr.index('L1 Wavefronts Shared'); continue
    if hdr is None or len(r) < len(hdr) - 5: continue
    if r[0]:
        cur = r[0]; lines[cur][3] = r[1]; continue
    try:
        i = float(r[ie] or 0); s = float(r[samp] or 0); w = float(r[wf] or 0)
    except ValueError:
        continue
    lines[cur][0] += i; lines[cur][1] += w; lines[cur][2] += s
    m = re.match(r'\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?', r[3])
    op = m.group(2) if m else '?'
    if op in ('LDS', 'STS') and m.group(3): op += m.group(3)
    ops[op][0] += i; ops[op][1] += w; ops[op][2] += s
ti = sum(v[0] for v in ops.values()); tw = sum(v[1] for v in ops.values()); ts = sum(v[2] for v in ops.values()) or 1
print(f"total warp instructions {ti:.4g}, shared wavefronts {tw:.4g}, stall samples {ts:.0f}")
print("-- opcodes")
for k, v in sorted(ops.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{k:14s} inst {v[0]:10.4g} {100*v[0]/ti:5.1f}%  wf {v[1]:10.4g}  stall {100*v[2]/ts:5.1f}%")
print("-- lines")
for k, v in sorted(lines.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{k:>5} inst {v[0]:10.4g} {100*v[0]/ti:5.1f}%  wf {v[1]:10.4g} stall {100*v[2]/ts:5.1f}%  {v[3].strip()[:80]}")
