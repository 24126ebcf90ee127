mkdir -p gpurun_out
CRUM_FUSED=1 timeout 400 ncu --set full --clock-control none -k regex:"k_fused_compare" -s 3 -c 1 -o gpurun_out/prof_fused python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu_f.log 2>&1
timeout 400 ncu --set full --clock-control none -k regex:"k_detect_hash" -s 3 -c 1 -o gpurun_out/prof_hash4k python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --mode hash --page 4096 > gpurun_out/ncu_h.log 2>&1
tail -1 gpurun_out/ncu_f.log gpurun_out/ncu_h.log
