# fence-free grid barrier in the small kernel: small-path parity, C1 lines x2, stamps
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_edges.py -q -k "small or every_path or edge or c1" 2>&1 | tail -1
O=gpurun_out/r03w; mkdir -p $O
for i in 1 2; do
timeout 300 python bench.py --config c1 --steps 200 --warmup 20 --no-cpu-baseline > $O/c1_$i.json 2> $O/c1_$i.err
python -c "import json; d=json.load(open('$O/c1_$i.json')); print(d['value'], d['ms_per_step'], d['call_latency']['cold_us'], d['call_latency']['warm_us'], d['call_latency']['kernel_us'], d['parity']['ok'])"
done
bash tools/gpu_r02_c1_stamps.sh 2>&1 | tail -16
