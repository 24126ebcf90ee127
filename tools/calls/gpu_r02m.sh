mkdir -p gpurun_out/r02m
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_soak.py tests/test_gpu_lazy.py tests/test_gpu_persist.py -q --timeout 600 2>&1 | tail -4
for m in compare tracked hash; do
  timeout 600 python bench.py --config c1 --mode $m --no-cpu-baseline > gpurun_out/r02m/c1_$m.json 2> gpurun_out/r02m/c1_$m.err
  python - gpurun_out/r02m/c1_$m.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], 'value', d['value'], 'us/step', round(d['ms_per_step']*1e3,1), 'e2e us', round(d['e2e']['ms_per_step']*1e3,1), 'dev us', round(d['device_phase']['ms_per_step']*1e3,1), 'kernel', d['roofline']['kernel'], d['roofline']['avg_launch_ms'], 'launches', d['gpu_launches'], 'parity', d['parity'].get('ok'))
PY
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "crum_checkpoint_gather_device/" --nvtx-include "crum_checkpoint_gather/" -c 60 --csv --log-file gpurun_out/r02m/launches_c1.csv python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r02m/c2.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/r02m/c2.json').read().strip().splitlines()[-1]);print('c2', d['value'], d['step']['frac'], d['device_phase'], d['parity']['ok'])"
