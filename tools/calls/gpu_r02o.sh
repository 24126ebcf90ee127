mkdir -p gpurun_out/r02o
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -k "hash" --timeout 600 2>&1 | tail -2
for rep in 1 2; do
for cfg in "--config c2 --page 65536" "--config c2 --page 2097152" "--config c4"; do
  tag=$(echo $cfg | tr -d ' -' )
  timeout 900 python bench.py $cfg --mode hash --no-cpu-baseline > gpurun_out/r02o/h_${tag}_$rep.json 2>/dev/null
  python - gpurun_out/r02o/h_${tag}_$rep.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d['roofline']; dp=d['device_phase']
print(sys.argv[1], 'value', d['value'], 'kernel', r['avg_launch_ms'], 'frac', r['frac'], 'dev', dp['value'], dp['frac'], 'parity', d['parity'].get('ok'))
PY
done
done
