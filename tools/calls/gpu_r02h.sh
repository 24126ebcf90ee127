mkdir -p gpurun_out/r02h
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_zenc -s 2 -c 1 -o gpurun_out/r02h/zenc_hpgmg3 python bench.py --config c2 --compress --content hpgmg --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
