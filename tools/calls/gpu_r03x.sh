# small kernel detect item size A/B: 1 KiB (log2 2), 2 KiB (1), 512 B (3)
O=gpurun_out/r03x; mkdir -p $O
run() {
  python -c "import __graft_entry__ as g; g.build()"
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -q -k "small or every_path" 2>&1 | tail -1
  for i in 1 2; do
    timeout 300 python bench.py --config c1 --steps 200 --warmup 20 --no-cpu-baseline --no-e2e > $O/il$1_$i.json 2> $O/il$1_$i.err
    python -c "import json; d=json.load(open('$O/il$1_$i.json')); print('items log2 $1', d['value'], d['ms_per_step'], d['call_latency']['cold_us'], d['call_latency']['warm_us'], d['call_latency']['kernel_us'], d['parity']['ok'])"
  done
}
run 2
for v in 1 3; do
  sed -i "s/constexpr uint32_t kSmallItemsLog2 = [0-9];/constexpr uint32_t kSmallItemsLog2 = $v;/" paper_1808_00117_b200/csrc/crum_internal.cuh
  run $v
done
