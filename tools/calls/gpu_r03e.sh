# mapped-store rule (serial <= 2 MiB, single pass 2-16 MiB): parity, then the C2 sweep (+ 1 %)
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q 2>&1 | tail -2
O=gpurun_out/r03e
mkdir -p $O
for mode in compare hash; do
for pg in 65536 2097152; do
 for d in 0.0 0.01 0.1 0.5 1.0; do
  f=$O/c2_${mode}_${pg}_${d}.json
  timeout 600 python bench.py --config c2 --mode $mode --page $pg --dirty $d --no-cpu-baseline > $f 2> ${f%.json}.err
  python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']; e=d['e2e']
print('$mode $pg $d', 'value', d['value'], 'ms', d['ms_per_step'], 'step frac', d['step']['frac'], 'kernel', r['frac'], 'dev', d['device_phase']['frac'], 'e2e', e['value'], 'restore', d['restore']['value'], d['restore']['link_frac'], 'parity', d['parity']['ok'])" 2>&1 | tail -1
 done
done
done
