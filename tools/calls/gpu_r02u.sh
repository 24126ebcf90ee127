# A/B: TMA hash kernels with 2 compute warps, 16 KiB rounds, 5 CTAs/SM
mkdir -p gpurun_out/r02u
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
one() {
  for cfg in "--config c2 --page 65536" "--config c2 --page 2097152" "--config c4"; do
    tag=$(echo $cfg | tr -d ' -' )
    timeout 900 python bench.py $cfg --mode hash --no-cpu-baseline --no-e2e > gpurun_out/r02u/$1_$tag.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/r02u/$1_$tag.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$1 $tag', 'kernel', r['avg_launch_ms'], 'frac', r['frac'], 'dev', d['device_phase']['frac'], 'parity', d['parity']['ok'])"
  done
}
one base
sed -i 's/constexpr int kTmaCompute = 4; /constexpr int kTmaCompute = 2; /; s/constexpr int kTmaCtasPerSm = 3; /constexpr int kTmaCtasPerSm = 5; /' paper_1808_00117_b200/csrc/kernels_detect.cu
grep -n "constexpr int kTmaCompute\|constexpr int kTmaCtasPerSm" paper_1808_00117_b200/csrc/kernels_detect.cu
python -c "from paper_1808_00117_b200 import build as b; b.build(force=True)" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "hash" --timeout 600 2>&1 | tail -1
one c2w5
