# compressed pinned gathers from 64 MiB ranges: parity, C2 lines x2, trace
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_compress.py -q -x 2>&1 | tail -1
O=gpurun_out/r03t; mkdir -p $O
for i in 1 2; do
for c in random half hpgmg; do
  timeout 400 python bench.py --config c2 --compress --content $c --no-cpu-baseline --no-e2e > $O/z_${c}_$i.json 2> $O/z_${c}_$i.err
  python -c "import json; d=json.load(open('$O/z_${c}_$i.json')); print('$c', d['value'], d['ms_per_step'], d['parity']['ok'])"
done
done
timeout 300 python tools/trace_e2e.py 65536 0.1 --compress > $O/trace_random.txt 2>&1
