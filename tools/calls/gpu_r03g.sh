# mapped split ranges + restored ring/D2H compressed pipeline: parity; d=1% lines; compressed ramp A/B
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_compress.py -q 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -20
O=gpurun_out/r03g; mkdir -p $O
for cfg in "compare 2097152" "hash 65536" "hash 2097152" "compare 65536"; do set -- $cfg
  for d in 0.0 0.01; do
  f=$O/c2_$1_$2_$d.json
  timeout 600 python bench.py --config c2 --mode $1 --page $2 --dirty $d --no-cpu-baseline > $f 2> ${f%.json}.err
  python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$1 $2 $d', 'value', d['value'], 'ms', d['ms_per_step'], 'step frac', d['step']['frac'], 'e2e', d['e2e']['value'], 'parity', d['parity']['ok'])" 2>&1 | tail -1
  done
done
for c in random half hpgmg; do
  timeout 400 python bench.py --config c2 --compress --content $c --steps 20 --warmup 5 --no-cpu-baseline > $O/c2z_$c.json 2> $O/c2z_$c.err
  python -c "import json; d=json.load(open('$O/c2z_$c.json')); print('ramp $c', d['value'], d['parity']['ok'])"
done
sed -i 's/constexpr uint32_t kZFirstUnits = 256;/constexpr uint32_t kZFirstUnits = 4096;/' paper_1808_00117_b200/csrc/crum_internal.cuh
python -c "import __graft_entry__ as g; g.build()"
for c in random half hpgmg; do
  timeout 400 python bench.py --config c2 --compress --content $c --steps 20 --warmup 5 --no-cpu-baseline > $O/c2z_noramp_$c.json 2> $O/c2z_noramp_$c.err
  python -c "import json; d=json.load(open('$O/c2z_noramp_$c.json')); print('noramp $c', d['value'], d['parity']['ok'])"
done
