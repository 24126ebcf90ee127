set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q 2>&1 | tail -3
mkdir -p gpurun_out/r02y
for i in 1 2; do timeout 300 python bench.py --config c1 --steps 200 --warmup 20 > gpurun_out/r02y/c1_$i.json 2>gpurun_out/r02y/c1_$i.err; tail -c 600 gpurun_out/r02y/c1_$i.json; done
bash tools/gpu_r02x.sh
