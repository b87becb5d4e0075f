python -c "import __graft_entry__ as g; g.build()" || exit 1
for d in 0 1 128 129; do echo "== debug=$d"; SNN_TRACE_DEBUG=$d timeout 300 python scripts/trace.py 3 0 2>&1 | grep -v "^{" | tail -3; done > gpurun_out/exp.log 2>&1
cat gpurun_out/exp.log
