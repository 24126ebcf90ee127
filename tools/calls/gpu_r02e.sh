mkdir -p gpurun_out/r02e
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for c in random half hpgmg; do
  timeout 600 python bench.py --config c2 --compress --content $c > gpurun_out/r02e/c2_z_$c.json 2> gpurun_out/r02e/c2_z_$c.err
  python - gpurun_out/r02e/c2_z_$c.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], 'value', d['value'], 'step frac', d['step']['frac'], 'comp', d.get('compression'), 'dev', d['device_phase']['value'], 'restore', d['restore']['value'], 'parity', d['parity'].get('ok'))
PY
done
timeout 600 python bench.py --config c2 --content hpgmg > gpurun_out/r02e/c2_hpgmg.json 2> gpurun_out/r02e/c2_hpgmg.err
python -c "import json;d=json.loads(open('gpurun_out/r02e/c2_hpgmg.json').read().strip().splitlines()[-1]);print('plain hpgmg', d['value'], d['parity'].get('ok'))"
timeout 900 python bench.py --compress --content hpgmg > gpurun_out/r02e/c4_z_hpgmg.json 2> gpurun_out/r02e/c4_z_hpgmg.err
python - gpurun_out/r02e/c4_z_hpgmg.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], 'value', d['value'], 'comp', d.get('compression'), 'restore', d['restore'], 'parity', d['parity'])
PY
tail -3 gpurun_out/r02e/*.err
