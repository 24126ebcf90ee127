python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_compress.py -q 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -30
mkdir -p gpurun_out/r03f
for c in random half hpgmg; do timeout 300 python tools/trace_e2e.py 65536 0.1 --compress --content $c > gpurun_out/r03f/trace_$c.txt 2>&1; done
for c in random half hpgmg; do
  timeout 400 python bench.py --config c2 --compress --content $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r03f/c2z_$c.json 2> gpurun_out/r03f/c2z_$c.err; echo "z $c rc=$?"
done
