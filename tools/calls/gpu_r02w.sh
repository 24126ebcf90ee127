mkdir -p gpurun_out/r02w
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1800 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_persist.py -q --timeout 600 2>&1 | tail -3
for cfg in "--config c2 --dirty 0.0" "--config c2 --dirty 0.01" "--config c2" "--config c2 --mode hash --page 2097152 --dirty 0.0" "--config c4"; do
  tag=$(echo $cfg | tr -d ' -' )
  timeout 900 python bench.py $cfg --no-cpu-baseline --no-e2e > gpurun_out/r02w/$tag.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02w/$tag.json').read().strip().splitlines()[-1]);s=d['step'];print('$tag', 'value', d['value'], 'ms', d['ms_per_step'], 'step frac', s['frac'], 'ideal', s['ideal_ms'], 'parity', d['parity']['ok'])"
done
