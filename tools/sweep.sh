#!/bin/bash
# tools/sweep.sh <out dir> -- run ON THE GPU BOX: one bench line per BASELINE.json config other
# than the default (configs 1, 2, 3; config 5 sweep points), each as its own bench.py run.
OUT=${1:-gpurun_out/sweep}
mkdir -p $OUT
run() {   # run <name> <bench args...>
  local n=$1; shift
  timeout 900 python bench.py "$@" > $OUT/$n.log 2>&1
  tail -1 $OUT/$n.log > $OUT/bench_$n.json
  python -c "import json,sys; d=json.load(open('$OUT/bench_$n.json')); print('$n', d['config'].get('prims'), d['config'].get('grid_res'), round(d['ms_per_step'],3), '%.4g' % d['value'], d.get('e2e',{}).get('value'))" 2>/dev/null || { echo "$n failed"; tail -3 $OUT/$n.log; }
}
run config1 --config 1 --steps 20 --warmup 5
run config2 --config 2 --steps 20 --warmup 5
run config3 --config 3 --steps 10 --warmup 3 --no-cpu-baseline
run config5_1M_1024 --config 5 --segments 1000000 --grid 1024 --no-cpu-baseline --no-finalize
run config5_5M_2048 --config 5 --segments 5000000 --grid 2048 --no-cpu-baseline --no-finalize
run config5_10M_4096 --config 5 --segments 10000000 --grid 4096 --no-cpu-baseline --no-finalize
run config5_10M_8192 --config 5 --segments 10000000 --grid 8192 --no-cpu-baseline --no-finalize --no-e2e
run config5_15M_8192 --config 5 --segments 15000000 --grid 8192 --no-cpu-baseline --no-finalize --no-e2e --steps 3
