#!/bin/bash
# Full oracle solve of BASELINE config C4 (N = 327,680) on the GPU box's host cores
# (CPU only; ~2.5 h on 16 threads).  Writes gpurun_out/oracle_C4.json, which is copied
# to tests/golden/ after review.  Calls only oracle/ and bipb_inputs/.
set -u
mkdir -p gpurun_out
lscpu > gpurun_out/c4_golden_lscpu.txt
python -c "import oracle; oracle.build(force=True)"
( time python tests/make_oracle_golden.py C4 --out=gpurun_out ) > gpurun_out/c4_golden.log 2>&1
echo "rc=$?" >> gpurun_out/c4_golden.log
tail -5 gpurun_out/c4_golden.log
