set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
for C in 0 4096; do
timeout 600 python bench.py --steps 3000 --warmup 500 --slice-width $C --no-cpu-baseline --no-e2e > gpurun_out/bench_C$C.log 2>&1; echo bench=$?
done
ncu --set full --clock-control none --import-source on -k regex:k_slice -s 1500 -c 1 -o gpurun_out/prof_slice_v5 python bench.py --steps 1000 --warmup 1000 --no-cpu-baseline --no-e2e --phase-steps 10 > gpurun_out/ncu_slice_v5.log 2>&1
