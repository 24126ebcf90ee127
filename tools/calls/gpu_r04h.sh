# C4 with HPGMG-like content: plain vs compressed images
O=gpurun_out/r04h; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py --content hpgmg --steps 10 --warmup 3 --no-cpu-baseline > $O/c4_hpgmg.json 2> $O/c4_hpgmg.err; echo "plain rc=$?"
timeout 900 python bench.py --content hpgmg --compress --steps 10 --warmup 3 --no-cpu-baseline > $O/c4_hpgmg_z.json 2> $O/c4_hpgmg_z.err; echo "z rc=$?"
for f in c4_hpgmg c4_hpgmg_z; do python -c "import json; d=json.load(open('$O/$f.json')); print('$f', d['value'], d['ms_per_step'], d['step']['frac'], d.get('compression',{}).get('ratio'), d['parity'].get('ok'), d['parity'].get('why'))"; done
tail -3 $O/c4_hpgmg_z.err
