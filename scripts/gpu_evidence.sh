# Round evidence of the default step (BASELINE config 3, ahead step graph):
# GPU tests, smoke, the driver's bench command and a long bench, the oracle arm,
# the ncu launch list of the bench command (cold-cache, serialised: shares),
# one --set full capture of each step kernel, and the builder's timing.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_driver.json 2> gpurun_out/bench_driver.err; echo bench_driver=$?
timeout 900 python bench.py --steps 10000 --warmup 1000 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_default=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 300 python scripts/build_only.py 3 3 > gpurun_out/build_times.txt 2>&1; cat gpurun_out/build_times.txt
python -c "import bench; print(bench.source_sha())" > gpurun_out/full_cur.sha
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_front|k_deliver|k_flush" -s 9000 -c 300 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 200 --warmup 20 --settle 3000 --no-cpu-baseline --no-e2e --no-ktime > gpurun_out/ncu_launch.log 2>&1
echo launches=$?
NCU_FLAGS=0 NCU_STEPS=3100 NSKIP=9000 NCOUNT=3 KREGEX="k_front|k_deliver|k_flush" bash scripts/gpu_ncu.sh
timeout 600 python bench.py --steps 10000 --warmup 1000 --history-bits 128 --no-cpu-baseline > gpurun_out/bench_h128.json 2> gpurun_out/bench_h128.err; echo bench_h128=$?
