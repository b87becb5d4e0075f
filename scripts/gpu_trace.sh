python -c "import __graft_entry__ as g; g.build()"
for C in 0 2048 512; do echo "== C=$C"; python scripts/trace.py 3 $C; done > gpurun_out/trace.log 2>&1
