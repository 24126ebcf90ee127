# end-of-session correctness: sanitizer workload, full pytest -m gpu, soak seeds
bash tools/gpu_round_check.sh
CRUM_SOAK_SEEDS=3-22 timeout 2400 python -m pytest tests/test_gpu_soak.py -q -m gpu 2>&1 | tail -2
