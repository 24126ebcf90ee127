# adaptive compressed chunks: parity + C2 / C4 lines
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_compress.py tests/test_gpu_persist.py tests/test_gpu_lazy.py -q -x 2>&1 | tail -1
O=gpurun_out/r04l; mkdir -p $O
for c in random half hpgmg; do
  timeout 400 python bench.py --config c2 --compress --content $c --no-cpu-baseline > $O/c2z_$c.json 2> $O/c2z_$c.err
  python -c "import json; d=json.load(open('$O/c2z_$c.json')); print('c2 $c', d['value'], d['ms_per_step'], d['compression']['ratio'], d['parity']['ok'])"
done
timeout 900 python bench.py --content hpgmg --compress --steps 10 --warmup 3 --no-cpu-baseline > $O/c4_hpgmg_z.json 2> $O/c4_hpgmg_z.err
python -c "import json; d=json.load(open('$O/c4_hpgmg_z.json')); print('c4 hpgmg z', d['value'], d['ms_per_step'], d['compression']['ratio'])"
