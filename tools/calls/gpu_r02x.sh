cp paper_1808_00117_b200/csrc/kernels_image.cu /tmp/ki_orig.cu
python tools/trace_small_patch.py
python -c "from paper_1808_00117_b200 import build as b; b.build(force=True)" 2>&1 | tail -3
timeout 300 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep "small:" | tail -12
