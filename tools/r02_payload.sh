#!/bin/bash
# GPU payload run beside the C4 oracle golden (tools/c4_golden_box.sh): test suite with a few
# OpenMP threads for the oracle checks, FP64 peak probes, bench, one full ncu capture of the
# symmetric kernel (CSV exports only: gpurun_out is capped at 64 MiB with the golden's products).
# Usage: bash tools/r02_payload.sh TAG [tests|bench|ncu|peak ...]
set -u
TAG=${1:-r02}; shift || true
WHAT=${*:-"tests peak bench ncu"}
O=gpurun_out/$TAG
mkdir -p $O
for w in $WHAT; do
  case $w in
    tests)
      OMP_NUM_THREADS=${PAYLOAD_OMP:-4} timeout ${TEST_TIMEOUT:-2300} python -m pytest ${PYTEST_SEL:-tests} -m gpu -q \
        -p no:cacheprovider --timeout 1200 -rfEs > $O/pytest_gpu.txt 2>&1
      tail -30 $O/pytest_gpu.txt ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -3 $O/smoke.txt ;;
    peak)
      tools/fp64_peak > $O/fp64_peak.jsonl 2>&1; tools/dmma_probe > $O/dmma_probe.jsonl 2>&1 ;;
    bench)
      timeout 900 python bench.py --no-cpu-baseline --precond-steps 0 > $O/bench.json 2> $O/bench.err
      tail -c 3000 $O/bench.json ;;
    ncu)
      timeout 600 ncu --set full --clock-control none --import-source on -k regex:^sym_kernel -s 1 -c 1 \
        -o /tmp/prof_sym_$TAG python tools/profile_driver.py C4 2 > $O/ncu_sym.log 2>&1
      ncu -i /tmp/prof_sym_$TAG.ncu-rep --page raw --csv > $O/prof_sym_raw.csv 2>&1
      ncu -i /tmp/prof_sym_$TAG.ncu-rep --page source --csv > $O/prof_sym_source.csv 2>&1
      ncu -i /tmp/prof_sym_$TAG.ncu-rep --page source --csv --print-source sass > $O/prof_sym_sass.csv 2>&1
      ncu -i /tmp/prof_sym_$TAG.ncu-rep --page details --csv > $O/prof_sym_details.csv 2>&1
      ls -la $O ;;
    tune)
      python tools/tune_matvec.py run C4 3 > $O/tune_sym_C4.jsonl 2> $O/tune_sym_C4.err; cat $O/tune_sym_C4.jsonl
      python tools/tune_matvec.py runbatch C4 > $O/tune_batch_C4.jsonl 2> $O/tune_batch_C4.err; cat $O/tune_batch_C4.jsonl ;;
    sanitize)
      for t in memcheck racecheck synccheck initcheck; do
        timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_driver.py > $O/sanitize_$t.txt 2>&1
        tail -3 $O/sanitize_$t.txt
      done ;;
    configs)
      for c in C1 C2 C3; do
        timeout 600 python bench.py --config $c --e2e-steps 0 --no-cpu-baseline --paper-tol-steps 1 > $O/bench_$c.json 2> $O/bench_$c.err
        tail -c 400 $O/bench_$c.json
      done ;;
    shards)
      timeout 900 python tools/shard_scaling.py C4 > $O/shard_scaling_C4.jsonl 2>&1; cat $O/shard_scaling_C4.jsonl ;;
    energy)
      python tools/tune_energy.py run C4 20 > $O/tune_energy_C4.jsonl 2> $O/tune_energy_C4.err; cat $O/tune_energy_C4.jsonl
      python tools/tune_energy.py run C3 50 > $O/tune_energy_C3.jsonl 2> $O/tune_energy_C3.err; cat $O/tune_energy_C3.jsonl ;;
    cycle)
      timeout 900 python -m pytest tests/test_gpu_cycle.py -m gpu -q -p no:cacheprovider -rfEs > $O/pytest_cycle.txt 2>&1
      tail -3 $O/pytest_cycle.txt
      for gm in 0 1 2; do
        BIPB_GRAPHS=$gm timeout 600 python tools/gmres_overhead.py C1 C2 C3 > $O/gmres_overhead_g$gm.txt 2>&1
        cat $O/gmres_overhead_g$gm.txt
      done ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
        python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --precond-steps 0 > /dev/null 2>&1 ;;
  esac
done
