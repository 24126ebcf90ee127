mkdir -p gpurun_out/r02l
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_persist.py tests/test_gpu_multirank.py tests/test_gpu_edges.py -q --timeout 600 2>&1 | tail -4
for m in compare hash; do
  timeout 600 python bench.py --config c1 --mode $m --no-cpu-baseline > gpurun_out/r02l/c1_$m.json 2> gpurun_out/r02l/c1_$m.err
  python - gpurun_out/r02l/c1_$m.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], 'value', d['value'], 'us/step', round(d['ms_per_step']*1e3,1), 'e2e us', round(d['e2e']['ms_per_step']*1e3,1), 'dev us', round(d['device_phase']['ms_per_step']*1e3,1), 'launches', d['gpu_launches'], 'parity', d['parity'].get('ok'))
PY
done
bash tools/gpu_r02k.sh
