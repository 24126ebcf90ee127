mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_edges.py tests/test_gpu_parity.py -q --timeout 600 -x 2>&1 | tail -15 > gpurun_out/r02b_pytest.txt
cat gpurun_out/r02b_pytest.txt
timeout 900 python bench.py > gpurun_out/r02b_c4.json 2> gpurun_out/r02b_c4.err; tail -c 4000 gpurun_out/r02b_c4.json; tail -5 gpurun_out/r02b_c4.err
timeout 600 python bench.py --config c2 > gpurun_out/r02b_c2.json 2> gpurun_out/r02b_c2.err; tail -c 600 gpurun_out/r02b_c2.json; tail -5 gpurun_out/r02b_c2.err
timeout 600 python bench.py --impl reference > gpurun_out/r02b_ref.json 2>&1; tail -c 1500 gpurun_out/r02b_ref.json
