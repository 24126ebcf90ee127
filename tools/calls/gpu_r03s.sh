# two alternating copy streams in the ring path: parity of pinned paths, C2 / C4 lines, trace
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -q -x -k "gather or deferred or capacity or mapped or every_path or full_size" 2>&1 | tail -1
O=gpurun_out/r03s; mkdir -p $O
for i in 1 2; do
for cfg in "compare 65536" "hash 65536" "compare 2097152"; do set -- $cfg
  timeout 400 python bench.py --config c2 --mode $1 --page $2 --dirty 0.1 --no-cpu-baseline > $O/c2_$1_$2_$i.json 2> $O/c2_$1_$2_$i.err
  python -c "import json; d=json.load(open('$O/c2_$1_$2_$i.json')); print('c2 $1 $2', d['value'], d['ms_per_step'], d['step']['frac'], d['parity']['ok'])"
done
done
timeout 600 python bench.py > $O/c4.json 2> $O/c4.err
python -c "import json; d=json.load(open('$O/c4.json')); print('c4', d['value'], d['ms_per_step'], d['step']['frac'], d['parity']['ok'])"
timeout 300 python tools/trace_e2e.py 65536 0.1 > $O/trace.txt 2>&1
