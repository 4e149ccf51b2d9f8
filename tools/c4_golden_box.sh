#!/bin/bash
# Full oracle solve of BASELINE config C4 (N = 327,680) on the GPU box's host cores, spread over
# several GPU-box calls: every GMRES product is kept (oracle.gmres_checkpointed), in /tmp on the
# box (survives a box reuse) and merged back under gpurun_out/c4_store/ (moved to tools/c4_store/
# here, which travels with the next snapshot).  CPU only; calls only oracle/ and bipb_inputs/.
# Usage: bash tools/c4_golden_box.sh LIMIT_S [payload command...]
# The payload (GPU work that needs little CPU) runs in the foreground meanwhile.
set -u
LIMIT=${1:-3300}; shift || true
STORE=/tmp/bipb_c4_store
mkdir -p gpurun_out/c4_store $STORE/C4_m20
[ -d tools/c4_store/C4_m20 ] && cp -n tools/c4_store/C4_m20/*.npy $STORE/C4_m20/ 2>/dev/null
ls $STORE/C4_m20 > /tmp/c4_before.txt
lscpu > gpurun_out/c4_golden_lscpu.txt
python -c "import oracle; oracle.build(force=True)"
( OMP_NUM_THREADS=${C4_THREADS:-15} timeout $LIMIT python tests/make_oracle_golden.py C4 --out=gpurun_out \
    --store=$STORE; echo "rc=$?" ) > gpurun_out/c4_golden.log 2>&1 &
GP=$!
if [ $# -gt 0 ]; then bash -c "$*"; echo "payload rc=$?"; fi
wait $GP
for f in $(ls $STORE/C4_m20); do grep -qx "$f" /tmp/c4_before.txt || cp $STORE/C4_m20/$f gpurun_out/c4_store/; done
ls $STORE/C4_m20 | wc -l
tail -4 gpurun_out/c4_golden.log
