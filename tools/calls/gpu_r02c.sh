mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_edges.py tests/test_gpu_parity.py -q --timeout 600 2>&1 | tail -15 > gpurun_out/r02c_pytest.txt
cat gpurun_out/r02c_pytest.txt
timeout 900 python bench.py > gpurun_out/r02c_c4.json 2> gpurun_out/r02c_c4.err; tail -c 300 gpurun_out/r02c_c4.json; tail -5 gpurun_out/r02c_c4.err
