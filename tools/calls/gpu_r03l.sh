python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "mapped and tracked" 2>&1 | grep -E "^E |Error|assert|passed|failed" | head -20
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -q -k "hash_single or fusable_hash or (mapped and hash)" 2>&1 | grep -E "^E |Error|passed|failed" | head -20
O=gpurun_out/r03l; mkdir -p $O
for d in 0.1 0.5 1.0; do
  timeout 400 python bench.py --config c2 --mode hash --page 65536 --dirty $d --no-cpu-baseline > $O/hash64k_$d.json 2> $O/hash64k_$d.err
  python -c "import json; d=json.load(open('$O/hash64k_$d.json')); print('$d', d['value'], d['step']['frac'], d['roofline']['kernel'], d['roofline']['frac'], d['device_phase'], d['parity']['ok'])"
done
