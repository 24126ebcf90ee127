mkdir -p gpurun_out/end
python -c "import __graft_entry__ as g; g.build()"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/end/default.json 2> gpurun_out/end/default.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/end/reference.json 2> gpurun_out/end/reference.err; echo "ref rc=$?"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/end/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
