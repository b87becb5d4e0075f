python -c "import __graft_entry__ as g; g.build()"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 200 -c 60 --csv --log-file gpurun_out/launches_v1.csv python bench.py --steps 40 --warmup 40 --no-cpu-baseline --no-e2e --phase-steps 10 > gpurun_out/ncu_launch_v1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stdp -s 20 -c 2 -o gpurun_out/prof_stdp_v1 python bench.py --steps 30 --warmup 30 --no-cpu-baseline --no-e2e --phase-steps 5 > gpurun_out/ncu_stdp_v1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_deliver -s 20 -c 2 -o gpurun_out/prof_deliver_v1 python bench.py --steps 30 --warmup 30 --no-cpu-baseline --no-e2e --phase-steps 5 > gpurun_out/ncu_deliver_v1.log 2>&1
ls -la gpurun_out
