mkdir -p gpurun_out/r02g
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_compress.py -q --timeout 600 2>&1 | tail -3
for c in random half hpgmg; do
  timeout 600 python bench.py --config c2 --compress --content $c --no-cpu-baseline > gpurun_out/r02g/c2_z_$c.json 2> gpurun_out/r02g/c2_z_$c.err
  python - gpurun_out/r02g/c2_z_$c.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
c=d.get('compression') or {}
print(sys.argv[1], 'value', d['value'], 'step frac', d['step']['frac'], 'ratio', c.get('ratio'), 'packed_ms', c.get('detect_to_last_chunk_packed_ms'), 'dev', d['device_phase']['value'], 'restore', d['restore']['value'], 'parity', d['parity'].get('ok'))
PY
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "crum_checkpoint_gather/" -c 40 --csv --log-file gpurun_out/r02g/launches_z_hpgmg.csv python bench.py --config c2 --compress --content hpgmg --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu1 rc=$?"
