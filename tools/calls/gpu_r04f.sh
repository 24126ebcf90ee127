python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -q -k "mapped or every_path or gather or deferred or capacity" 2>&1 | tail -1
O=gpurun_out/r04f; mkdir -p $O
for d in 0.02 0.03; do
  timeout 400 python bench.py --config c2 --dirty $d --no-cpu-baseline --no-e2e > $O/c2_$d.json 2> $O/c2_$d.err
  python -c "import json; d=json.load(open('$O/c2_$d.json')); print('c2 $d', d['value'], d['ms_per_step'], d['step']['frac'], d['parity']['ok'])"
done
