mkdir -p gpurun_out/r02r
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1800 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_compress.py -q --timeout 600 2>&1 | tail -4
for d in 0.1 0.5 1.0; do
  timeout 600 python bench.py --config c2 --dirty $d --no-cpu-baseline --no-e2e > gpurun_out/r02r/c2_$d.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02r/c2_$d.json').read().strip().splitlines()[-1]);print('c2 d=$d', 'value', d['value'], 'dev', d['device_phase']['value'], d['device_phase']['frac'], 'kernel', d['roofline']['kernel'], d['roofline']['frac'], 'parity', d['parity']['ok'])"
done
