python -c "import __graft_entry__ as g; g.build()" >/dev/null || exit 1
# K = 16: steps 1501..1503 (1503 is a batch step, 1503 % 16 == 15)
SNN_TRACE_KW='{"flush_period": 16}' SNN_TRACE_T0=1501 timeout 300 python scripts/trace.py 3 0 2>&1 | grep -v "^{\|^front"
