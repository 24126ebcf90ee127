# Page-group TMA hash detect: parity (auto, forced NP=4, forced NP=2) and A/B timing
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -m gpu -x 2>&1 | tail -1
CRUM_HASH_NP=4 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_soak.py -q -m gpu -x 2>&1 | tail -1
CRUM_HASH_NP=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "hash or mixed or full_size or gather" 2>&1 | tail -1
mkdir -p gpurun_out/pair
for pg in 65536 2097152; do for v in "" CRUM_HASH_NP=2 CRUM_HASH_TMA1=1; do
  env $v timeout 120 python bench.py --mode hash --page $pg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pair/o.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/pair/o.json').read().strip().splitlines()[-1]);print($pg,'$v',d['value'],d['roofline']['achieved'],d['roofline']['frac'])"
done; done
for v in "" CRUM_HASH_NP=2; do
  env $v timeout 300 python bench.py --config c4 --mode hash --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pair/o.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/pair/o.json').read().strip().splitlines()[-1]);print('c4','$v',d['value'],d['roofline']['achieved'],d['roofline']['frac'])"
done
