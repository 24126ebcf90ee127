# C1 latency anatomy: bench c1, c1_latency, ncu --set full of k_small_ckpt
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r03h; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "mapped or small" 2>&1 | tail -1
timeout 300 python bench.py --config c1 --steps 200 --warmup 20 --no-cpu-baseline > $O/c1.json 2> $O/c1.err; echo "c1 rc=$?"
timeout 300 python tools/c1_latency.py > $O/c1_latency.txt 2>&1; echo "lat rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_small_ckpt --launch-skip 30 -c 1 -o $O/c1_small python bench.py --config c1 --steps 5 --warmup 30 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
