# state check: build, GPU parity tests, default bench line, phase trace
set -x
python -c "import __graft_entry__ as g; g.build()"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
cat MEASURED_PEAKS.json > gpurun_out/peaks.json 2>/dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench=$?
cat gpurun_out/bench_full.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
