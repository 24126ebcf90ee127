mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_compress.py -q --timeout 600 > gpurun_out/r02d_pytest.txt 2>&1
grep -n "Error\|error\|FAILED\|passed\|failed" gpurun_out/r02d_pytest.txt | head -30

