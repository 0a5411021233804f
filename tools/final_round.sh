#!/bin/bash
# tools/final_round.sh <out dir> -- run ON THE GPU BOX at the end of a round: the bench lines
# committed under profiles/, the GPU test log, then the ncu evidence (tools/profile_round.sh).
OUT=$1
mkdir -p $OUT
python bench.py > $OUT/bench.log 2>&1; tail -1 $OUT/bench.log > $OUT/bench.json
python bench.py --impl reference > $OUT/ref.log 2>&1; tail -1 $OUT/ref.log > $OUT/bench_reference.json
python bench.py --sampled 8 --no-cpu-baseline > $OUT/s8.log 2>&1; tail -1 $OUT/s8.log > $OUT/bench_sampled8.json
python bench.py --config 3 --no-cpu-baseline > $OUT/c3.log 2>&1; tail -1 $OUT/c3.log > $OUT/bench_config3.json
python bench.py --config 2 --distance hist --no-cpu-baseline > $OUT/h2.log 2>&1; tail -1 $OUT/h2.log > $OUT/bench_hist_config2.json
python bench.py --distance hist --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-finalize > $OUT/h4.log 2>&1; tail -1 $OUT/h4.log > $OUT/bench_hist_config4.json
python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1
bash tools/profile_round.sh $OUT/prof
