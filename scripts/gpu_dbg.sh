python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python scripts/dbg_rw.py > gpurun_out/dbg_rw.log 2>&1; echo rc=$?
tail -40 gpurun_out/dbg_rw.log
