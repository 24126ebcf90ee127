# TMA hash-detect ring depth / CTAs-per-SM sweep (C2 hash, 2 MiB and 64 KiB pages)
mkdir -p gpurun_out/sw
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -m gpu -x 2>&1 | tail -2
for pg in 2097152 65536; do
  for st in 2 3 4; do for c in 1 2 3; do
    CRUM_TMA_STAGES=$st CRUM_TMA_CTAS=$c timeout 120 python bench.py --mode hash --page $pg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw/h_${pg}_${st}_${c}.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/sw/h_${pg}_${st}_${c}.json').read().strip().splitlines()[-1]);print($pg,$st,$c,d['value'],d['roofline']['achieved'],d['roofline']['frac'],d['device_phase']['frac'])"
  done; done
done
