O=gpurun_out/r04b; mkdir -p $O
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/c3.json 2> $O/c3.err; echo "c3 rc=$?"
timeout 300 python bench.py --config c1 --steps 200 --warmup 20 --no-cpu-baseline > $O/c1.json 2> $O/c1.err; echo "c1 rc=$?"
for f in c3 c1; do python -c "import json; d=json.load(open('$O/$f.json')); r=d['roofline']; print('$f', d['value'], r['frac'], r['read_stream_GBs'], d['parity']['ok'])"; done
