python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r04m; mkdir -p $O
for i in 1 2 3; do
  timeout 400 python bench.py --config c2 --compress --content random --no-cpu-baseline --no-e2e > $O/r_$i.json 2> $O/r_$i.err
  python -c "import json; d=json.load(open('$O/r_$i.json')); print('c2 random', d['value'], d['ms_per_step'])"
done
timeout 400 python bench.py --config c2 --no-cpu-baseline --no-e2e > $O/plain.json 2> $O/plain.err
python -c "import json; d=json.load(open('$O/plain.json')); print('c2 plain', d['value'], d['ms_per_step'])"
