mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -x 2>&1 | tail -3
for a in "--config c1" "" "--config c1 --mode hash" "--mode tracked"; do
 for env in "" "CRUM_NO_GRAPH=1"; do
  env $env timeout 300 python bench.py --no-cpu-baseline --no-e2e $a > gpurun_out/g.json 2>&1
  python - <<PY
import json
d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1]); r=d['roofline']
print("$a $env", 'value', d['value'], 'ms', d['ms_per_step'], r['kernel'], r['frac'], 'launches', d['gpu_launches'])
PY
 done
done
