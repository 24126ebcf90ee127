# A/B: single-pass kernel occupancy (launch bounds) on C2 at d = 0.1 and 1
mkdir -p gpurun_out/r02q
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
one() {
  for d in 0.1 1.0; do
    timeout 600 python bench.py --config c2 --fused --dirty $d --no-cpu-baseline --no-e2e > gpurun_out/r02q/$1_$d.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/r02q/$1_$d.json').read().strip().splitlines()[-1]);print('$1 d=$d', 'dev', d['device_phase']['value'], d['device_phase']['frac'], 'kernel', d['roofline']['frac'], 'parity', d['parity']['ok'])"
  done
}
one lb_default
for b in 6 8; do
  sed -i "s/__global__ void __launch_bounds__(kFusedThreads[^)]*) k_fused_compare/__global__ void __launch_bounds__(kFusedThreads, $b) k_fused_compare/" paper_1808_00117_b200/csrc/kernels_image.cu
  python -c "from paper_1808_00117_b200 import build as b; b.build(force=True)" 2>&1 | tail -2
  one lb_$b
done
