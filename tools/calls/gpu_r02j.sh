# round-2 evidence: every GPU test, smoke, default bench (C4), reference arm,
# NVTX-filtered launch list of the default bench, ncu --set full of the C4 detect
mkdir -p gpurun_out/r02j
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
timeout 2700 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02j/pytest.txt 2>&1; tail -8 gpurun_out/r02j/pytest.txt
timeout 900 python bench.py > gpurun_out/r02j/default.json 2> gpurun_out/r02j/default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r02j/reference.json 2> gpurun_out/r02j/reference.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "crum_checkpoint_gather/" --nvtx-include "crum_checkpoint_gather_device/" -c 300 --csv --log-file gpurun_out/r02j/launches_default.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02j/ncu_bench.json 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "crum_checkpoint_gather_device/" -k regex:k_detect_compare -c 1 -o gpurun_out/r02j/c4_detect_compare python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu full rc=$?"
