# single-pass kernel: L2 prefetch of the next segment A/B (on / off)
O=gpurun_out/r04c; mkdir -p $O
run() {
  python -c "import __graft_entry__ as g; g.build()"
  timeout 600 python -m pytest tests/test_gpu_variants.py -q -x -k "fusable" 2>&1 | tail -1
  for d in 0.01 0.1 1.0; do
    timeout 400 python bench.py --config c2 --dirty $d --fused --no-cpu-baseline --no-e2e > $O/pf$1_$d.json 2> $O/pf$1_$d.err
    python -c "import json; d=json.load(open('$O/pf$1_$d.json')); r=d['roofline']; print('pf$1 $d', d['value'], d['ms_per_step'], r['kernel'], r['frac'], d['device_phase']['frac'], d['parity']['ok'])"
  done
}
run on
sed -i 's/constexpr bool kFusedPrefetch = true;/constexpr bool kFusedPrefetch = false;/' paper_1808_00117_b200/csrc/kernels_image.cu
run off
