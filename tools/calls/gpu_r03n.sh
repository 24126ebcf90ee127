# hash page-pair kernel: L2 prefetch cursor A/B (kPairPrefetch 4 / 0 / 2 / 8) on C2 64 KiB and C4 hash
O=gpurun_out/r03n; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "hash" 2>&1 | tail -1
run() {
  for d in 0.0 0.1; do
    timeout 400 python bench.py --config c2 --mode hash --page 65536 --dirty $d --no-cpu-baseline --no-e2e > $O/pf$1_c2_$d.json 2> $O/pf$1_c2_$d.err
    python -c "import json; d=json.load(open('$O/pf$1_c2_$d.json')); r=d['roofline']; print('pf$1 c2 $d', r['kernel'], r['frac'], r['avg_launch_ms'], d['device_phase']['frac'], d['parity']['ok'])"
  done
  timeout 600 python bench.py --config c4 --mode hash --no-cpu-baseline --no-e2e > $O/pf$1_c4.json 2> $O/pf$1_c4.err
  python -c "import json; d=json.load(open('$O/pf$1_c4.json')); r=d['roofline']; print('pf$1 c4', r['kernel'], r['frac'], r['avg_launch_ms'], d['device_phase']['frac'], d['parity']['ok'])"
}
run 4
for v in 0 2 8; do
  sed -i "s/constexpr uint32_t kPairPrefetch = [0-9]*;/constexpr uint32_t kPairPrefetch = $v;/" paper_1808_00117_b200/csrc/kernels_detect.cu
  python -c "import __graft_entry__ as g; g.build()"
  run $v
done
