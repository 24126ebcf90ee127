# C1 latency study: default graph path vs fused single-pass vs no graph; launch list
mkdir -p gpurun_out/c1
python -c "import __graft_entry__ as g; g.build()"
for v in default CRUM_FUSED=1 CRUM_NO_GRAPH=1 "CRUM_FUSED=1 CRUM_NO_GRAPH=1"; do
  if [ "$v" = default ]; then e=""; else e="$v"; fi
  env $e timeout 120 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/c1/out.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/c1/out.json').read().strip().splitlines()[-1]);print('$v', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['avg_launch_ms'], d['e2e']['value'], d['e2e']['ms_per_step'], d['gpu_launches'])"
done
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/c1/launch.csv python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
