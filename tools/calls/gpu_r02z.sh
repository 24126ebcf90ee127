python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q 2>&1 | tail -2
python tools/c1_latency.py 2>&1 | grep "^{"
mkdir -p gpurun_out/r02z
for i in 1 2; do timeout 300 python bench.py --config c1 --steps 200 --warmup 20 > gpurun_out/r02z/c1_$i.json 2>gpurun_out/r02z/c1_$i.err; done
