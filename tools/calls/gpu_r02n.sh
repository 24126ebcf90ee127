mkdir -p gpurun_out/r02n
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_small_ckpt -s 8 -c 1 -o gpurun_out/r02n/small_c1 python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
