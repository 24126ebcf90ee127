mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -x 2>&1 | tail -2
timeout 300 python bench.py --config c2 --page 4096 --mode hash --no-cpu-baseline --no-e2e > gpurun_out/q1.json 2>&1
CRUM_FUSED=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/q2.json 2>&1
timeout 300 python bench.py --mode hash --no-cpu-baseline --no-e2e > gpurun_out/q3.json 2>&1
for f in gpurun_out/q1.json gpurun_out/q2.json gpurun_out/q3.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print(d['config']['workload'], 'value', d['value'], 'ms', d['ms_per_step'], r['kernel'], r['achieved'], r['frac'], 'dev', d['device_phase']['frac'])"; done
