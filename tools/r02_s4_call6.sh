#!/bin/bash
# r02 session 4: device-side GMRES cycles (BIPB_GRAPHS=2) -- parity test and the per-solve A/B.
set -u
mkdir -p gpurun_out/s4f
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4f/build.txt 2>&1; tail -3 gpurun_out/s4f/build.txt
OMP_NUM_THREADS=16 bash tools/r02_payload.sh s4f cycle
