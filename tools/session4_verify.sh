set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s4_env.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > gpurun_out/s4_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4_pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/s4_bench.json 2> gpurun_out/s4_bench.err; echo bench=$?
tail -3 gpurun_out/s4_pytest_gpu.log; cat gpurun_out/s4_bench.json
