for cv in 25 -1 100 50; do
SNN_DELIVER_CARVEOUT=$cv timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('carveout $cv ms/step', d['ms_per_step'], d['roofline']['phase_ms_per_step'])"
done
