python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 compute-sanitizer --tool memcheck --show-backtrace no python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize.log 2>&1; echo rc=$?
head -60 gpurun_out/sanitize.log
