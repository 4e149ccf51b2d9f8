#!/usr/bin/env bash
# One GPU session's measurement set (run under gpurun from the repo root):
#   bench (JSON line), launch list under ncu, one full ncu capture of the symmetric matvec
#   kernel, one of the source + energy kernels, and the sym kernel's traffic.
# Usage: tools/round_profile.sh TAG        -> gpurun_out/{bench,launches,prof_sym,prof_src_en}_TAG*
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p "$OUT"
export OMP_PROC_BIND=close OMP_PLACES=cores
timeout 900 python bench.py > "$OUT/bench_$TAG.json" 2> "$OUT/bench_$TAG.err"
cat "$OUT/bench_$TAG.json"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches_$TAG.csv" \
  python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:^sym_kernel -s 1 -c 1 \
  -o "$OUT/prof_sym_$TAG" python tools/profile_driver.py C4 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 0 -c 2 \
  -o "$OUT/prof_src_en_$TAG" python tools/profile_driver.py C4 0 --all > /dev/null 2>&1
for r in sym src_en; do
  [ -f "$OUT/prof_${r}_$TAG.ncu-rep" ] && ncu -i "$OUT/prof_${r}_$TAG.ncu-rep" --page raw --csv > "$OUT/prof_${r}_$TAG.csv" 2>/dev/null
done
ls -la "$OUT" | grep "$TAG"
