# A/B: host pipeline lookahead (ranges enqueued ahead of the host): 2 vs all
mkdir -p gpurun_out/r02v
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
one() {
  for cfg in "--config c2 --dirty 0.0" "--config c2 --dirty 0.01" "--config c2" "--config c2 --mode hash --page 2097152" "--config c4"; do
    tag=$(echo $cfg | tr -d ' -' )
    timeout 900 python bench.py $cfg --no-cpu-baseline --no-e2e > gpurun_out/r02v/$1_$tag.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/r02v/$1_$tag.json').read().strip().splitlines()[-1]);s=d['step'];print('$1 $tag', 'value', d['value'], 'ms', d['ms_per_step'], 'step frac', s['frac'], 'ideal', s['ideal_ms'], 'parity', d['parity']['ok'])"
  done
}
one a2
sed -i 's/    constexpr uint32_t kAhead = 2;/    constexpr uint32_t kAhead = 1000;/' paper_1808_00117_b200/csrc/runtime.cu
python -c "from paper_1808_00117_b200 import build as b; b.build(force=True)" 2>&1 | tail -2
one aall
