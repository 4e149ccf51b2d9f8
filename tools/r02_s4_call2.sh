#!/bin/bash
# r02 session 4, call N: C4 oracle golden products on the box's host cores (store carried in
# tools/c4_store/C4_m20) while a GPU payload runs; if the golden completes, the golden parity tests.
# Usage: TAG=s4b LIMIT=3000 PAYLOAD="sanitize configs" bash tools/r02_s4_call2.sh
set -u
TAG=${TAG:-s4b}
mkdir -p gpurun_out/$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/$TAG/build.txt 2>&1
C4_THREADS=${C4_THREADS:-14} PAYLOAD_OMP=2 bash tools/c4_golden_box.sh ${LIMIT:-3000} \
  "bash tools/r02_payload.sh $TAG ${PAYLOAD:-sanitize}" > gpurun_out/$TAG/golden_call.txt 2>&1
tail -8 gpurun_out/$TAG/golden_call.txt
if [ -f gpurun_out/oracle_C4.json ]; then
  cp gpurun_out/oracle_C4.json tests/golden/oracle_C4.json
  OMP_NUM_THREADS=16 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider \
    -k "golden" -rfEs > gpurun_out/$TAG/pytest_golden.txt 2>&1
  tail -5 gpurun_out/$TAG/pytest_golden.txt
fi
