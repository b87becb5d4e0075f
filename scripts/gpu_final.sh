# the round's final evidence: gpu_evidence.sh + every BASELINE config
bash scripts/gpu_evidence.sh
bash scripts/gpu_configs_r02.sh
