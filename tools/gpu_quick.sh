mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -x 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/q1.json 2>&1
CRUM_NO_DPIPE=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/q2.json 2>&1
timeout 300 python bench.py --mode hash --no-cpu-baseline --no-e2e > gpurun_out/q3.json 2>&1
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q4.json 2>&1
for f in gpurun_out/q1.json gpurun_out/q2.json gpurun_out/q3.json gpurun_out/q4.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print(d['config']['workload'], 'value', d['value'], 'ms', d['ms_per_step'], r['kernel'], r['achieved'], r['frac'], 'dev', d['device_phase']['frac'])"; done
