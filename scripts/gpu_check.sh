set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
python scripts/trace.py 3 0 > gpurun_out/trace.log 2>&1
timeout 600 python bench.py --steps 3000 --warmup 500 --no-cpu-baseline --no-e2e > gpurun_out/bench_C0.log 2>&1; echo bench=$?
ncu --set full --clock-control none --import-source on -k regex:"k_stdp" -s 1000 -c 1 -o gpurun_out/prof_v13 python bench.py --steps 1000 --warmup 1000 --no-cpu-baseline --no-e2e --phase-steps 10 > gpurun_out/ncu_v13.log 2>&1
