mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_lazy.py tests/test_gpu_persist.py tests/test_gpu_parity.py -q --timeout 300 -x 2>&1 | tail -15
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/l1.json 2>&1
tail -c 1800 gpurun_out/l1.json
