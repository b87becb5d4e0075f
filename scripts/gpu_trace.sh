python -c "import __graft_entry__ as g; g.build()"
python scripts/trace.py 3 0 > gpurun_out/trace.log 2>&1
python scripts/trace.py 3 2048 >> gpurun_out/trace.log 2>&1
