set -x
nvidia-smi -L
nproc
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout 600 python bench.py --steps 2000 --warmup 200 > gpurun_out/bench.log 2>&1; echo bench=$?
