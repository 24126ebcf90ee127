# end-of-round correctness: full pytest -m gpu, then the extended soak
python -c "import __graft_entry__ as g; g.build()"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -2
bash tools/gpu_soak_long.sh
