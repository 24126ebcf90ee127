# hash 2 MiB full-size parity, repeated (the TMA ring release race), then the TMA sweep
run() { for i in 1 2 3 4 5 6 7 8; do timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "full_size_parity and 2097152-1" 2>&1 | grep -E "^E  |passed|failed" | head -2 | tr '\n' ' '; echo; done; }
python -c "import __graft_entry__ as g; g.build()"
echo "== current"; run
mkdir -p gpurun_out/sw
for pg in 2097152 65536; do
  for st in 2 3; do for c in 2 3; do
    CRUM_TMA_STAGES=$st CRUM_TMA_CTAS=$c timeout 120 python bench.py --mode hash --page $pg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw/h_${pg}_${st}_${c}.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/sw/h_${pg}_${st}_${c}.json').read().strip().splitlines()[-1]);print($pg,$st,$c,d['value'],d['roofline']['achieved'],d['roofline']['frac'],d['device_phase']['frac'])"
  done; done
done
