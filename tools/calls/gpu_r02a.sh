set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -3
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -30 > gpurun_out/r02a_pytest.txt
cat gpurun_out/r02a_pytest.txt
timeout 600 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; tail -c 3000 gpurun_out/r02a_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02a_ref.json 2>&1; tail -c 1500 gpurun_out/r02a_ref.json
nvidia-smi --query-gpu=name,memory.total --format=csv; nproc; free -g; numactl -H 2>/dev/null | head -5; lscpu | grep -E "Model name|NUMA"
