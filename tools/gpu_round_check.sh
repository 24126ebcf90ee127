# correctness check of every kernel: the sanitizer workload (every kernel vs the oracle) and pytest -m gpu.
# (compute-sanitizer is closed on the GPU pool since round 2: runs under it left GPUs needing a reset;
#  the round-1 / early round-2 sanitizer logs are in profiles/sanitizer/.)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python tools/sanitize_run.py 2>&1 | tail -3
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -x 2>&1 | tail -4
