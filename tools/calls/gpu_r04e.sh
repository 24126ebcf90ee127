# mapped single pass up to 64 MiB payloads (compare-only): C2 at 2 / 5 % vs the ring (CFG_NO_MAPPED via --no-mapped unavailable: compare with r04d)
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r04e; mkdir -p $O
for d in 0.02 0.05 0.07; do
  timeout 400 python bench.py --config c2 --dirty $d --no-cpu-baseline --no-e2e > $O/c2_$d.json 2> $O/c2_$d.err
  python -c "import json; d=json.load(open('$O/c2_$d.json')); r=d['roofline']; print('c2 $d', d['value'], d['ms_per_step'], d['step']['frac'], r['kernel'], d['parity']['ok'])"
done
sed -i 's/constexpr uint64_t kMappedFusedPayload = 64ull << 20;/constexpr uint64_t kMappedFusedPayload = 16ull << 20;/' paper_1808_00117_b200/csrc/runtime.cu
python -c "import __graft_entry__ as g; g.build()"
for d in 0.02 0.05 0.07; do
  timeout 400 python bench.py --config c2 --dirty $d --no-cpu-baseline --no-e2e > $O/ring_c2_$d.json 2> $O/ring_c2_$d.err
  python -c "import json; d=json.load(open('$O/ring_c2_$d.json')); r=d['roofline']; print('ring c2 $d', d['value'], d['ms_per_step'], d['step']['frac'], r['kernel'], d['parity']['ok'])"
done
