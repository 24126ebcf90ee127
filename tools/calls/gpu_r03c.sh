# encoder fast-path rounds + unrolled pack: parity, launch times, C2 compressed lines
mkdir -p gpurun_out/r03c
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_compress.py -x -q 2>&1 | tail -2
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_z --csv --log-file gpurun_out/r03c/zenc_launches.csv python tools/trace_e2e.py 65536 0.1 --compress --content hpgmg > /dev/null 2>&1; echo "ncu rc=$?"
for c in random hpgmg; do timeout 300 python tools/trace_e2e.py 65536 0.1 --compress --content $c > gpurun_out/r03c/trace_$c.txt 2>&1; done
for c in random half hpgmg; do
  timeout 400 python bench.py --config c2 --compress --content $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r03c/c2z_$c.json 2> gpurun_out/r03c/c2z_$c.err; echo "z $c rc=$?"
done
