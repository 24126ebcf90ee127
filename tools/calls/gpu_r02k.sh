# A/B: 64 KiB hash pages on the TMA page-pair kernel (kBigHashLog2 = 16)
# vs the warp-per-page kernel (kBigHashLog2 = 17)
mkdir -p gpurun_out/r02k
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for cfg in "--config c2 --page 65536" "--config c4"; do
  tag=$(echo $cfg | tr -d ' -' )
  timeout 900 python bench.py $cfg --mode hash --no-cpu-baseline > gpurun_out/r02k/b16_$tag.json 2>/dev/null
done
sed -i 's/constexpr uint32_t kBigHashLog2 = 16;/constexpr uint32_t kBigHashLog2 = 17;/' paper_1808_00117_b200/csrc/crum_internal.cuh
python -c "from paper_1808_00117_b200 import build as b; b.build(force=True)" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "hash" --timeout 600 2>&1 | tail -2
for cfg in "--config c2 --page 65536" "--config c4"; do
  tag=$(echo $cfg | tr -d ' -' )
  timeout 900 python bench.py $cfg --mode hash --no-cpu-baseline > gpurun_out/r02k/b17_$tag.json 2>/dev/null
done
for f in gpurun_out/r02k/*.json; do python - $f <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d['roofline']; dp=d['device_phase']
print(sys.argv[1], 'value', d['value'], 'kernel', r['kernel'], r['avg_launch_ms'], 'frac', r['frac'], 'dev', dp['value'], dp['frac'], 'parity', d['parity'].get('ok'))
PY
done
