mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compress.py tests/test_gpu_lazy.py -q --timeout 300 -x 2>&1 | tail -3
for pg in 65536 2097152; do
 for env in "" "CRUM_HASH_NO_TMA=1"; do
  env $env timeout 300 python bench.py --mode hash --page $pg --no-cpu-baseline --no-e2e > gpurun_out/t.json 2>&1
  python - <<PY
import json
d=json.loads(open('gpurun_out/t.json').read().strip().splitlines()[-1]); r=d['roofline']
print("$pg $env", 'value', d['value'], 'ms', d['ms_per_step'], r['kernel'], r['achieved'], r['frac'], 'dev', d['device_phase']['frac'])
PY
 done
done
env timeout 600 python bench.py --config c4 --mode hash --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/t.json 2>&1; tail -c 600 gpurun_out/t.json
