# Round-2 ncu evidence of the default step (BASELINE config 3, ahead step graph):
# (1) the launch list of the bench command (per-launch times, cold-cache and
#     serialised by ncu: shares, not absolutes), (2) one --set full capture of
#     each step kernel after the settle steps (graph nodes profiled one by one).
python -c "import __graft_entry__ as g; g.build()" || exit 1
python -c "import bench; print(bench.source_sha())" > gpurun_out/full_cur.sha
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_front|k_deliver|k_flush" -s 9000 -c 300 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 200 --warmup 20 --settle 3000 --no-cpu-baseline --no-e2e --no-ktime > gpurun_out/ncu_launch.log 2>&1
echo launches=$?
NCU_FLAGS=0 NCU_STEPS=3100 NSKIP=9000 NCOUNT=3 KREGEX="k_front|k_deliver|k_flush" bash scripts/gpu_ncu.sh
ls -la gpurun_out | head -20
