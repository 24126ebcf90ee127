# A/B: encoder hash-round unroll 4 (default) vs 8, C2 compressed
mkdir -p gpurun_out/r02s
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
one() {
  for c in random hpgmg; do
    timeout 600 python bench.py --config c2 --compress --content $c --no-cpu-baseline --no-e2e > gpurun_out/r02s/$1_$c.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/r02s/$1_$c.json').read().strip().splitlines()[-1]);c=d['compression'];print('$1 $c', 'value', d['value'], 'ratio', c['ratio'], 'packed_ms', c['detect_to_last_chunk_packed_ms'], 'parity', d['parity']['ok'])"
  done
}
one u4
sed -i 's/constexpr uint32_t kUnroll = 4;/constexpr uint32_t kUnroll = 8;/' paper_1808_00117_b200/csrc/kernels_zip.cu
python -c "from paper_1808_00117_b200 import build as b; b.build(force=True)" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_compress.py -q -x 2>&1 | tail -1
one u8
