#!/bin/bash
# tools/profile_round.sh <out dir> -- run ON THE GPU BOX: launch list with DRAM bytes of one
# bench step, and ncu --set full captures of the hot kernels, summarised in place (the
# .ncu-rep files are deleted after summarising so the directory stays small).
# Optional second argument: a space-separated list of kernels to capture (default: all).
OUT=$1
ONLY=${2:-}
mkdir -p $OUT
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-finalize"
$B > $OUT/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches.csv $B > $OUT/ncu_launch.log 2>&1
python3 tools/launch_traffic.py $OUT/launches.csv > $OUT/traffic.json
cap() {   # cap <kernel regex> <name> <command...>
  local k=$1 n=$2; shift 2
  if [ -n "$ONLY" ] && [[ " $ONLY " != *" $n "* ]]; then return; fi
  ncu --set full --clock-control none --import-source on -k regex:$k -s 0 -c 1 -o $OUT/$n "$@" > $OUT/ncu_$n.log 2>&1
  if [ -f $OUT/$n.ncu-rep ]; then
    python3 tools/ncu_summary.py $OUT/$n.ncu-rep "$n" > $OUT/$n.md
    ncu -i $OUT/$n.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null > $OUT/$n.src.csv
    { echo; echo "Top source lines (share of warp-stall samples, instructions executed):"; echo; echo '```';
      python3 tools/ncu_lines.py $OUT/$n.src.csv 15; echo '```'; } >> $OUT/$n.md
    rm -f $OUT/$n.ncu-rep $OUT/$n.src.csv
  fi
}
for k in k_sggxh_quad k_sggxh_half k_sggxh_warp k_fiber_emit k_bin_reduce_warp k_lod_prep_leaf; do cap $k $k $B; done
cap k_encode k_encode python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e
cap k_spline_emit k_spline_emit $B --sampled 8
cap k_fiber_density k_fiber_density python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e
cap k_sggxh_hist k_sggxh_hist python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-finalize --config 2 --distance hist
ls -la $OUT
