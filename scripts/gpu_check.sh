python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
python scripts/trace.py 3 0 > gpurun_out/trace_new.log 2>&1
python bench.py --steps 3000 --warmup 300 --no-cpu-baseline --no-e2e > gpurun_out/bench_new.json 2>&1
tail -n 3 gpurun_out/bench_new.json
