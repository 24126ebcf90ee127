# compressed gathers: chunk ramp (trace per chunk), parity tests, C2 lines per content
mkdir -p gpurun_out/r03a
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_compress.py -x -q 2>&1 | tail -2
for c in random hpgmg; do timeout 300 python tools/trace_e2e.py 65536 0.1 --compress --content $c > gpurun_out/r03a/trace_$c.txt 2>&1; done
for c in random half hpgmg; do
  timeout 400 python bench.py --config c2 --compress --content $c --steps 20 --warmup 5 > gpurun_out/r03a/c2z_$c.json 2> gpurun_out/r03a/c2z_$c.err; echo "z $c rc=$?"
done
timeout 400 python bench.py --config c2 --steps 20 --warmup 5 > gpurun_out/r03a/c2_plain.json 2> gpurun_out/r03a/c2_plain.err; echo "plain rc=$?"
