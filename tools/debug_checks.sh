#!/bin/bash
# tools/debug_checks.sh <out dir> -- run ON THE GPU BOX: builds the bounds-checked library
# (-DVOX_DEBUG -> paper_2604_13191_b200/libvox_dbg.so, separate objects) and runs the GPU test
# suite against it; every test also asserts that no check fired (tests/conftest.py). This
# stands in for compute-sanitizer, which is closed on the GPU pool.
OUT=${1:-gpurun_out/dbg}
mkdir -p $OUT
VOX_NVCC_EXTRA=-DVOX_DEBUG python - <<'PY'
import os
from paper_2604_13191_b200 import build as B
B.LIB = B.LIB.replace("libvox.so", "libvox_dbg.so")
B.OBJ = B.OBJ + "_dbg"
print(B.build(force=True))
PY
VOX_DEBUG_LIB=1 python -m pytest tests -m gpu -q -x "${@:2}" > $OUT/pytest_gpu_debug.txt 2>&1
echo "rc=$?"; tail -3 $OUT/pytest_gpu_debug.txt
