mkdir -p gpurun_out/sweep
python -c "import __graft_entry__ as g; g.build()"
for pg in 65536 2097152; do
 for d in 0.0 0.1 0.5 1.0; do
  timeout 600 python bench.py --page $pg --dirty $d --no-cpu-baseline > gpurun_out/sweep/c2_${pg}_${d}.json 2> gpurun_out/sweep/c2_${pg}_${d}.err
  python -c "
import json
d=json.loads(open('gpurun_out/sweep/c2_${pg}_${d}.json').read().strip().splitlines()[-1]); r=d['roofline']; e=d['e2e']
print('$pg $d', 'value', d['value'], 'ms', d['ms_per_step'], r['frac'], 'dev', d['device_phase']['frac'], 'e2e', e['value'], e.get('link_roofline'), 'restore', d['restore']['value'])" 2>&1 | tail -1
 done
done
