python -c "import __graft_entry__ as g; g.build()" || exit 1
for d in ${TRACE_DEBUGS:-none}; do
  if [ "$d" = none ]; then timeout 300 python scripts/trace.py 3 0 > gpurun_out/trace_$d.log 2>&1;
  else SNN_TRACE_DEBUG=$d timeout 300 python scripts/trace.py 3 0 > gpurun_out/trace_$d.log 2>&1; fi
  echo "== debug $d"; grep -E "^(front|stdp|deliver) " gpurun_out/trace_$d.log | tail -3
done
