# timing + whole-step DRAM traffic (device phase) for C1-C4, compare / hash,
# default vs the single-pass kernel (--fused)
mkdir -p gpurun_out/r02p
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
run() {  # tag, args...
  tag=$1; shift
  timeout 900 python bench.py "$@" --no-cpu-baseline > gpurun_out/r02p/$tag.json 2> gpurun_out/r02p/$tag.err
  alg=$(python -c "import json;d=json.loads(open('gpurun_out/r02p/$tag.json').read().strip().splitlines()[-1]);print(d['device_phase']['alg_bytes_per_step'])" 2>/dev/null)
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "crum_checkpoint_gather_device/" -c 80 --csv --log-file gpurun_out/r02p/${tag}_traffic.csv python bench.py "$@" --no-cpu-baseline --steps 3 --warmup 3 > /dev/null 2>&1
  python - gpurun_out/r02p/$tag.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d['roofline']; dp=d['device_phase']
print(sys.argv[1].split('/')[-1], 'value', d['value'], 'step', d['step']['frac'], 'kernel', r['kernel'], r['frac'], 'dev', dp['value'], dp['frac'], 'parity', d['parity'].get('ok'))
PY
  [ -n "$alg" ] && python tools/step_traffic.py gpurun_out/r02p/${tag}_traffic.csv $alg 3 | head -1
}
run c1_compare --config c1
run c2_compare_d01 --config c2
run c2_compare_d01_fused --config c2 --fused
run c2_compare_d1 --config c2 --dirty 1.0
run c2_compare_d1_fused --config c2 --dirty 1.0 --fused
run c2_hash64k_d01 --config c2 --mode hash
run c2_hash64k_d1 --config c2 --mode hash --dirty 1.0
run c4_compare --config c4
run c4_compare_fused --config c4 --fused
run c4_hash --config c4 --mode hash
run c3_compare --config c3 --restore-full
