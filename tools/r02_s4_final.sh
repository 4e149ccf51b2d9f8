#!/bin/bash
# r02 session 4, verification call on the committed tree: build, smoke, the whole GPU suite (no
# CPU contention), the default bench, the launch list, and one full ncu capture of the source and
# energy pair kernels (CSV exports into gpurun_out/$TAG).
set -u
TAG=${TAG:-s4e}
O=gpurun_out/$TAG
mkdir -p $O
export OMP_PROC_BIND=close OMP_PLACES=cores
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
OMP_NUM_THREADS=16 timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=30 -rfEs \
  > $O/pytest_gpu.txt 2>&1; tail -4 $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 600 $O/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -c 2 \
  -o /tmp/prof_src_en_$TAG python tools/profile_driver.py C4 0 --all > $O/ncu_src_en.log 2>&1
ncu -i /tmp/prof_src_en_$TAG.ncu-rep --page raw --csv > $O/prof_src_en_raw.csv 2>&1
ls -la $O
