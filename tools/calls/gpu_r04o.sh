# extended soak on the final code: 60 soak seeds, 10x full-size hash parity, 5x every kernel path, 5x mapped + compress
python -c "import __graft_entry__ as g; g.build()"
CRUM_SOAK_SEEDS=3-62 timeout 3000 python -m pytest tests/test_gpu_soak.py -q -m gpu 2>&1 | tail -1
for i in 1 2 3 4 5 6 7 8 9 10; do timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "full_size or repeatable" 2>&1 | tail -1; done
for i in 1 2 3 4 5; do timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_compress.py -q -m gpu 2>&1 | tail -1; done
for i in 1 2 3 4 5; do timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "mapped or small or synth" 2>&1 | tail -1; done
