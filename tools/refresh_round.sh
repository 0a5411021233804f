#!/bin/bash
# tools/refresh_round.sh <out dir> -- run ON THE GPU BOX: the default bench line and the launch
# list (with DRAM bytes) of one step, plus the density kernel capture (a subset of final_round.sh).
OUT=$1
mkdir -p $OUT/prof
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-finalize"
$B > $OUT/prof/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/prof/launches.csv $B > $OUT/prof/ncu_launch.log 2>&1
python3 tools/launch_traffic.py $OUT/prof/launches.csv > $OUT/prof/traffic.json
cp $OUT/prof/traffic.json profiles/r01_traffic.json   # bench.py reads roofline.traffic from here
python bench.py > $OUT/bench.log 2>&1; tail -1 $OUT/bench.log > $OUT/bench.json
n=k_fiber_density
ncu --set full --clock-control none --import-source on -k regex:$n -s 0 -c 1 -o $OUT/prof/$n \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/prof/ncu_$n.log 2>&1
python3 tools/ncu_summary.py $OUT/prof/$n.ncu-rep "$n" > $OUT/prof/$n.md
ncu -i $OUT/prof/$n.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null > $OUT/prof/$n.src.csv
{ echo; echo "Top source lines (share of warp-stall samples, instructions executed):"; echo; echo '```';
  python3 tools/ncu_lines.py $OUT/prof/$n.src.csv 15; echo '```'; } >> $OUT/prof/$n.md
rm -f $OUT/prof/$n.ncu-rep $OUT/prof/$n.src.csv
