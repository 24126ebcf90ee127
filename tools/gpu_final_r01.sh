mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build()"
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/final/$name.json 2> gpurun_out/final/$name.err; echo "$name rc=$?"; tail -c 300 gpurun_out/final/$name.json | head -c 300; echo; }
run c2_compare
run reference --impl reference
run c2_hash64k --mode hash --no-cpu-baseline
run c2_hash4k --mode hash --page 4096 --no-cpu-baseline --no-e2e
run c2_hash2m --mode hash --page 2097152 --no-cpu-baseline
run c2_compare2m --page 2097152 --no-cpu-baseline --no-e2e
run c2_tracked --mode tracked --no-cpu-baseline
run c2_zhalf --compress --content half --no-cpu-baseline
run c2_half --content half --no-cpu-baseline
run c1_compare --config c1 --no-cpu-baseline
run c3_compare --config c3 --steps 10 --warmup 3 --no-cpu-baseline
run c4_compare --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e
run c4_hash --config c4 --mode hash --steps 5 --warmup 3 --no-cpu-baseline --no-e2e
run c5_hash --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/final/torchrun1.json 2> gpurun_out/final/torchrun1.err; echo "torchrun rc=$?"
