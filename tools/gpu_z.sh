mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_compress.py -q --timeout 300 -x 2>&1 | tail -30
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lazy.py tests/test_gpu_persist.py -q --timeout 300 -x 2>&1 | tail -5
