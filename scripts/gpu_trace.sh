python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python scripts/trace.py 3 0 > gpurun_out/trace.log 2>&1; echo trace=$?
cat gpurun_out/trace.log
