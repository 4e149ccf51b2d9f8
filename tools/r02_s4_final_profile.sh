#!/bin/bash
# r02 session 4 end: the committed tree's launch list (default bench, W = 3, K = 1) and one full ncu
# capture each of the C4 symmetric product (exact sums, the bench's kernel) and the source + energy
# kernels; CSV exports into gpurun_out/s4z.
set -u
O=gpurun_out/s4z
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --paper-tol-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:^sym_kernel -s 1 -c 1 \
  -o /tmp/prof_sym_s4z python tools/profile_driver.py C4 2 > $O/ncu_sym.log 2>&1
ncu -i /tmp/prof_sym_s4z.ncu-rep --page raw --csv > $O/prof_sym_raw.csv 2>&1
ncu -i /tmp/prof_sym_s4z.ncu-rep --page details --csv > $O/prof_sym_details.csv 2>&1
ls -la $O
