mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for a in "--content half" "--content half --compress" "--compress" "--content half --compress --dirty 1.0"; do
  timeout 300 python bench.py --no-cpu-baseline $a > gpurun_out/z.json 2>&1
  python - <<PY
import json
d=json.loads(open('gpurun_out/z.json').read().strip().splitlines()[-1])
print("$a", 'value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], d['e2e']['ms_per_step'], 'img', d['config']['image_bytes_per_step'], d.get('compression'), 'restore', d['restore'], 'forked', d['forked']['pause_ms'])
PY
done
