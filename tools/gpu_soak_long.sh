# Extended correctness soak: 20 soak seeds, repeated full-size hash parity
# (the TMA ring race showed up there), repeated hash stress, all kernel variants
mkdir -p gpurun_out/soak
python -c "import __graft_entry__ as g; g.build()"
CRUM_SOAK_SEEDS=3-22 timeout 2400 python -m pytest tests/test_gpu_soak.py -q -m gpu 2>&1 | tail -2
for i in 1 2 3 4 5 6; do timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "full_size or repeatable" 2>&1 | tail -1; done
CRUM_HASH_TMA1=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "full_size or repeatable or straddle" 2>&1 | tail -1
CRUM_HASH_NO_TMA=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "full_size or repeatable or straddle" 2>&1 | tail -1
CRUM_COMPACT2=1 CRUM_SOAK_SEEDS=30-33 timeout 1200 python -m pytest tests/test_gpu_soak.py -q -m gpu 2>&1 | tail -1
CRUM_NO_GRAPH=1 CRUM_SOAK_SEEDS=40-43 timeout 1200 python -m pytest tests/test_gpu_soak.py -q -m gpu 2>&1 | tail -1
