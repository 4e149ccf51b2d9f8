#!/bin/bash
# Session 3 of r02: finish the C4 oracle golden (products carried in tools/c4_store), meanwhile the
# GPU-only tuning probes; then, if the golden completed, test the GPU solve against it.
set -u
mkdir -p gpurun_out/r02d
C4_THREADS=15 bash tools/c4_golden_box.sh 3000 "bash tools/r02_payload.sh r02d tune" > gpurun_out/r02d/golden_call.txt 2>&1
cat gpurun_out/r02d/golden_call.txt | tail -5
if [ -f gpurun_out/oracle_C4.json ]; then
  cp gpurun_out/oracle_C4.json tests/golden/oracle_C4.json
  OMP_NUM_THREADS=16 timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider \
    -k "golden" -rfEs > gpurun_out/r02d/pytest_golden.txt 2>&1
  tail -5 gpurun_out/r02d/pytest_golden.txt
fi
