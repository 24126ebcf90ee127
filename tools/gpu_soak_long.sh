# Extended correctness soak: 20 soak seeds, repeated full-size hash parity
# (the TMA ring race showed up there), every kernel path selected through
# crum_config (tests/test_gpu_variants.py), repeated.
mkdir -p gpurun_out/soak
python -c "import __graft_entry__ as g; g.build()"
CRUM_SOAK_SEEDS=3-22 timeout 2400 python -m pytest tests/test_gpu_soak.py -q -m gpu 2>&1 | tail -2
for i in 1 2 3 4 5 6; do timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "full_size or repeatable" 2>&1 | tail -1; done
for i in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_variants.py -q -m gpu 2>&1 | tail -1; done
