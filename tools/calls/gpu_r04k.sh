# compressed chunk size A/B: 16 MiB (shipped) vs 32 MiB vs 8 MiB
O=gpurun_out/r04k; mkdir -p $O
run() {
  python -c "import __graft_entry__ as g; g.build()"
  timeout 900 python -m pytest tests/test_gpu_compress.py -q -x 2>&1 | tail -1
  for c in random hpgmg; do
    timeout 400 python bench.py --config c2 --compress --content $c --no-cpu-baseline --no-e2e > $O/cu$1_c2_$c.json 2> $O/cu$1_c2_$c.err
    python -c "import json; d=json.load(open('$O/cu$1_c2_$c.json')); print('units $1 c2 $c', d['value'], d['ms_per_step'], d['parity']['ok'])"
  done
  timeout 900 python bench.py --content hpgmg --compress --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/cu$1_c4.json 2> $O/cu$1_c4.err
  python -c "import json; d=json.load(open('$O/cu$1_c4.json')); print('units $1 c4 hpgmg', d['value'], d['ms_per_step'])"
}
sed -i "s/constexpr uint32_t kZChunkUnits = [0-9]*;/constexpr uint32_t kZChunkUnits = 8192;/" paper_1808_00117_b200/csrc/crum_internal.cuh
run 8192
for v in 16384; do
  sed -i "s/constexpr uint32_t kZChunkUnits = [0-9]*;/constexpr uint32_t kZChunkUnits = $v;/" paper_1808_00117_b200/csrc/crum_internal.cuh
  run $v
done
