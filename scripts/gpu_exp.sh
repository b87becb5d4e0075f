python -c "import __graft_entry__ as g; g.build()" >/dev/null || exit 1
timeout 300 python scripts/trace.py 3 0 2>&1 | grep -v "^{" | tail -3
