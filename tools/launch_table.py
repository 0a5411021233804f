"""profiles/<tag>_launches.md from the traffic JSON of tools/launch_traffic.py (one bench step)."""
import json, sys
tag, src = sys.argv[1], sys.argv[2]
t = json.load(open(src))
tot = sum(v["ms"] for v in t.values())
rows = sorted(t.items(), key=lambda kv: -kv[1]["ms"])
print(f"# {tag} launch list (one step of config 4, `bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-finalize`)\n")
print(f"From `profiles/{tag}_launches.csv` (`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
      "dram__bytes_write.sum\n--clock-control none`; cold-cache, serialised launches: compare shares, not absolute "
      "times). `tools/launch_traffic.py` aggregates the last step.\n")
print("| kernel | launches | ms | share | DRAM GB (read + write) |\n|---|---|---|---|---|")
for k, v in rows:
    print(f"| `{k}` | {v['launches']} | {v['ms']:.3f} | {100 * v['ms'] / tot:.1f} % | {v['dram_bytes'] / 1e9:.2f} |")
print(f"| total | {sum(v['launches'] for v in t.values())} | {tot:.2f} | | "
      f"{sum(v['dram_bytes'] for v in t.values()) / 1e9:.1f} |")
