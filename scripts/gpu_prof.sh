python scripts/trace.py 3 0 > gpurun_out/trace.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_stdp|k_deliver" -s 3000 -c 2 -o gpurun_out/prof_v8 python bench.py --steps 1000 --warmup 1000 --no-cpu-baseline --no-e2e --phase-steps 10 > gpurun_out/ncu_v8.log 2>&1
