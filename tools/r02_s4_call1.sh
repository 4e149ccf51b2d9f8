#!/bin/bash
# r02 session 4, call 1: C4 oracle golden products on the box's host cores (continuing the local
# store in tools/c4_store/C4_m20) while the GPU payload runs: smoke, the whole GPU suite, the bench.
set -u
mkdir -p gpurun_out/s4a
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4a/build.txt 2>&1
C4_THREADS=14 PAYLOAD_OMP=2 bash tools/c4_golden_box.sh ${LIMIT:-3000} "bash tools/r02_payload.sh s4a smoke tests bench" \
  > gpurun_out/s4a/golden_call.txt 2>&1
tail -8 gpurun_out/s4a/golden_call.txt
