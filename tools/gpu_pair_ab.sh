# Page-group TMA hash detect: parity (default NP=2, forced NP=4) and timing
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_soak.py -q -m gpu -x 2>&1 | tail -1
CRUM_HASH_NP=4 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -m gpu -x 2>&1 | tail -1
for args in "--mode hash" "--mode hash --page 2097152" "--mode hash --config c4 --steps 5 --warmup 3" "--mode hash --config c3 --steps 5 --warmup 3"; do
  timeout 300 python bench.py --steps 20 --warmup 5 $args --no-cpu-baseline --no-e2e > /tmp/o.json 2>/dev/null
  python -c "import json;d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]);print('$args',d['value'],d['roofline']['achieved'],d['roofline']['frac'],d['device_phase']['frac'],d.get('parity',{}).get('ok'))"
done
