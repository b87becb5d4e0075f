# round evidence: GPU tests, full default bench line, reference (oracle) arm,
# ncu launch list of the bench command, one ncu --set full capture of the step kernels
set -x
python -c "import __graft_entry__ as g; g.build()"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 200 --warmup 20 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 3000 -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1000 --warmup 1000 --no-cpu-baseline --no-e2e --phase-steps 10 > gpurun_out/ncu_launch.log 2>&1
KREGEX="k_deliver|k_stdp|k_front" NCOUNT=3 NSKIP=4400 bash scripts/gpu_ncu.sh
ABL_STEPS=1000 bash scripts/gpu_ablation.sh > /dev/null 2>&1; cp gpurun_out/ablation.jsonl gpurun_out/ablation_round.jsonl
timeout 600 python bench.py --steps 3000 --warmup 300 --no-cpu-baseline --no-e2e --idx16 > gpurun_out/bench_idx16.json 2>/dev/null
