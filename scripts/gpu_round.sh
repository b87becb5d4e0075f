# round evidence: full default bench line, launch list, ncu full capture of the step kernels
set -x
python -c "import __graft_entry__ as g; g.build()"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 200 --warmup 20 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 3000 -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1000 --warmup 1000 --no-cpu-baseline --no-e2e --phase-steps 10 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_stdp|k_deliver|k_front" -s 3000 -c 3 -o gpurun_out/prof_round python bench.py --steps 1000 --warmup 1000 --no-cpu-baseline --no-e2e --phase-steps 10 > gpurun_out/ncu_round.log 2>&1
