#!/bin/bash
# tools/make_profiles.sh <src dir under gpurun_out> <round tag>  -> profiles/<tag>_*.{json,csv,md}
set -e
SRC=$1; TAG=$2
cp $SRC/bench.json profiles/${TAG}_bench.json
cp $SRC/launches.csv profiles/${TAG}_launches.csv
python3 tools/launches.py profiles/${TAG}_launches.csv k_fiber_bound > /tmp/l.txt
{ echo "# ${TAG} launch list (one step of config 4, from profiles/${TAG}_launches.csv)"; echo; echo '```'; cat /tmp/l.txt; echo '```'; } > profiles/${TAG}_launches.md
for k in sggxh_warp sggxh_quad fiber_emit; do
  if [ -f $SRC/$k.ncu-rep ]; then
    python3 tools/ncu_summary.py $SRC/$k.ncu-rep "$k (config 4, 10.28M segments, 4096^3)" > /tmp/k.md
    ncu -i $SRC/$k.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null > /tmp/k.csv
    { cat /tmp/k.md; echo; echo "Top source lines (share of warp-stall samples, instructions executed):"; echo; echo '```'; python3 tools/ncu_lines.py /tmp/k.csv 15; echo '```'; } > profiles/${TAG}_$k.md
  fi
done
ls profiles/
