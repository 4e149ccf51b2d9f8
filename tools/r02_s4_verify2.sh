#!/bin/bash
# r02 session 4: the small block shape (B = 128) and the new default-kernel rule -- whole GPU suite,
# smoke, C1/C2/C4 benches.
set -u
O=gpurun_out/${TAG:-s4m}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
OMP_NUM_THREADS=16 timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 -rfEs > $O/pytest_gpu.txt 2>&1
tail -20 $O/pytest_gpu.txt
for c in C1 C2 C3; do
  timeout 600 python bench.py --config $c --e2e-steps 0 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  python -c "import json; d=json.load(open('$O/bench_$c.json')); print('$c', d['value'], d['ms_per_step'], d['iterations'][-1], d.get('oracle_golden',{}).get('pass'))"
done
timeout 900 python bench.py > $O/bench_C4.json 2> $O/bench_C4.err
python -c "import json; d=json.load(open('$O/bench_C4.json')); print('C4', d['value'], d['ms_per_step'], d['e2e']['value'], d['oracle_golden']['pass'])"
