#!/usr/bin/env bash
# One GPU session validating the exact limb sums (bipb_set_sum_mode 1; csrc/bipb_exact.cuh):
#   exact-mode GPU tests, C4 bench in both sum modes, the exact kernel's DRAM traffic (ncu), and
#   the whole GPU suite with BIPB_SUM=fixed (every context starts in mode 0, the non-default).
# Usage (repo root, under gpurun): tools/exact_validate.sh TAG  -> gpurun_out/xv_TAG_*
set -u
TAG=${1:-s3}
OUT=gpurun_out
mkdir -p "$OUT"
P="$OUT/xv_${TAG}"
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_multirank.py -k "exact" -q -x \
  > "${P}_tests.log" 2>&1
echo "exit $?" >> "${P}_tests.log"
for m in fixed exact; do
  timeout 600 python bench.py --sum $m --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --precond-steps 0 \
    > "${P}_bench_$m.json" 2> "${P}_bench_$m.err"
done
timeout 300 env BIPB_SUM=exact ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:sym_kernel -s 1 -c 1 --csv python tools/profile_driver.py C4 2 \
  > "${P}_ncu_exact.csv" 2>&1
timeout 1500 env BIPB_SUM=fixed python -m pytest tests -m gpu -q -x > "${P}_suite_fixed.log" 2>&1
echo "exit $?" >> "${P}_suite_fixed.log"
tail -n 3 "${P}_tests.log" "${P}_suite_fixed.log"
cat "${P}_bench_fixed.json" "${P}_bench_exact.json" | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l); r = d['roofline']
    print(d['config'].get('sums'), d['value'], d['time_to_solution_s'], r['avg_launch_ms'], r['frac'])"
