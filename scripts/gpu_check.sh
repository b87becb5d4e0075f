timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
for D in 0 3; do
SNN_TRACE_DEBUG=$D python scripts/trace.py 3 0 > gpurun_out/trace_d$D.log 2>&1
done
timeout 600 python bench.py --steps 3000 --warmup 500 --no-cpu-baseline --no-e2e > gpurun_out/bench_C0.log 2>&1; echo bench=$?
