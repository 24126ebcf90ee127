mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err; tail -3 gpurun_out/bench_torchrun1.err; cat gpurun_out/bench_torchrun1.json
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_detect_compare|k_gather|k_compact_write|k_crc_meta" -s 8 -c 4 -o gpurun_out/prof_c2_compare python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu1.log 2>&1; tail -2 gpurun_out/ncu1.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_detect_hash_big" -s 3 -c 1 -o gpurun_out/prof_c2_hash64k python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --mode hash > gpurun_out/ncu2.log 2>&1; tail -2 gpurun_out/ncu2.log
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 150 --csv --log-file gpurun_out/launches_hash.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --mode hash > /dev/null 2>&1
ls -la gpurun_out | tail
