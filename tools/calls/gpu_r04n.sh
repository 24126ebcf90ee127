# compressed chunk cap 64 MiB (shipped) vs 128 MiB on C4 HPGMG-like
O=gpurun_out/r04n; mkdir -p $O
run() {
  python -c "import __graft_entry__ as g; g.build()"
  timeout 900 python bench.py --content hpgmg --compress --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/cap$1_c4.json 2> $O/cap$1_c4.err
  python -c "import json; d=json.load(open('$O/cap$1_c4.json')); print('cap $1 c4 hpgmg z', d['value'], d['ms_per_step'])"
}
run 16384
sed -i "s/constexpr uint32_t kZChunkUnits = 16384;/constexpr uint32_t kZChunkUnits = 32768;/" paper_1808_00117_b200/csrc/crum_internal.cuh
timeout 600 python -m pytest tests/test_gpu_compress.py -q -x 2>&1 | tail -1
run 32768
