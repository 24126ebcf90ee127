mkdir -p gpurun_out/r02t
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1800 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_edges.py -q --timeout 600 2>&1 | tail -3
for m in compare hash tracked; do
  timeout 600 python bench.py --config c1 --mode $m --no-cpu-baseline > gpurun_out/r02t/c1_$m.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02t/c1_$m.json').read().strip().splitlines()[-1]);print('c1 $m', 'value', d['value'], 'us/step', round(d['ms_per_step']*1e3,1), 'e2e us', d['e2e']['ms_per_step']*1e3, 'dev us', round(d['device_phase']['ms_per_step']*1e3,1), 'parity', d['parity']['ok'])"
done
