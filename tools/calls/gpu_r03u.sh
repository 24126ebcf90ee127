python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "pool_and_numa" 2>&1 | tail -1
O=gpurun_out/r03u; mkdir -p $O
for i in 1 2 3; do
  timeout 400 python bench.py --config c2 --dirty 0.1 --no-cpu-baseline --no-e2e > $O/c2_$i.json 2> $O/c2_$i.err
  python -c "import json; d=json.load(open('$O/c2_$i.json')); print('c2', d['value'], d['ms_per_step'], d['step']['frac'], d['step']['link_peak_GBs'], d['parity']['ok'])"
done
