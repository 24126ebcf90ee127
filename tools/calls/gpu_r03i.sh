# C1 single bitmap: small-path parity, c1 lines, latency
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r03i; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_edges.py -q -k "small or variants or edge or every_path" 2>&1 | tail -1
timeout 300 python bench.py --config c1 --steps 200 --warmup 20 --no-cpu-baseline > $O/c1.json 2> $O/c1.err; echo "c1 rc=$?"
python -c "import json; d=json.load(open('$O/c1.json')); print(d['value'], d['ms_per_step'], d['call_latency'], d['parity']['ok'])"
timeout 300 python tools/c1_latency.py > $O/c1_latency.txt 2>&1; echo "lat rc=$?"; grep "^{" $O/c1_latency.txt | head -4
