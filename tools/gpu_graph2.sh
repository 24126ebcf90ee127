mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -x 2>&1 | tail -2
for a in "--config c1" ""; do
 for env in "" "CRUM_NO_GRAPH=1"; do
  env $env timeout 300 python bench.py --no-cpu-baseline --no-e2e $a > gpurun_out/g.json 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$a $env', 'value', d['value'], 'ms', d['ms_per_step'], r['kernel'], r['frac'], 'launches', d['gpu_launches'])" 2>&1 | tail -1
 done
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c1.csv python bench.py --config c1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_compact_write|k_crc_meta|k_compact_count|k_gather|k_detect" -s 20 -c 5 -o gpurun_out/prof_c1 python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/n7.log 2>&1
