# batched synth: parity of the batched fill/writer, default line, plain launch list (-c 400)
O=gpurun_out/batch; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "synth" 2>&1 | tail -1
timeout 600 python bench.py > $O/default.json 2> $O/default.err; echo "default rc=$?"
python -c "import json; d=json.load(open('$O/default.json')); print(d['value'], d['ms_per_step'], d['step']['frac'], d['parity']['ok'], d['gpu_launches'], d['gpu_launches_synth'])"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
