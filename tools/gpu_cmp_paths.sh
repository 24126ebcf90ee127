mkdir -p gpurun_out
for cfg in c3 c4; do
  timeout 400 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/bf_$cfg.json 2>&1
  CRUM_NO_FUSED=1 timeout 400 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/bn_$cfg.json 2>&1
done
timeout 400 python bench.py --config c4 --mode hash --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/bh_c4.json 2>&1
timeout 400 python bench.py --config c2 --page 4096 --mode hash --no-cpu-baseline --no-e2e > gpurun_out/bh_c2_4k.json 2>&1
timeout 400 python bench.py --config c2 --page 4096 --no-cpu-baseline --no-e2e > gpurun_out/bf_c2_4k.json 2>&1
for f in gpurun_out/bf_*.json gpurun_out/bn_*.json gpurun_out/bh_*.json; do echo $f; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print(d['config']['workload'], 'value', d['value'], 'ms', d['ms_per_step'], r['kernel'], r['achieved'], r['frac'], 'dev', d['device_phase']['frac'])"; done
