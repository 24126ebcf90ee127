# Session-3 evidence: bench lines for every configuration, reference arm,
# launch lists and ncu --set full captures of the dominant kernels.
O=gpurun_out/r01c
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
run() { name=$1; shift; timeout 900 python bench.py "$@" > $O/$name.json 2> $O/$name.err; echo "$name rc=$?"; }
run c2_compare
run reference --impl reference
run c2_hash64k --mode hash --no-cpu-baseline
run c2_hash4k --mode hash --page 4096 --no-cpu-baseline --no-e2e
run c2_hash2m --mode hash --page 2097152 --no-cpu-baseline
run c2_compare2m --page 2097152 --no-cpu-baseline --no-e2e
run c2_tracked --mode tracked --no-cpu-baseline
run c2_zhalf --compress --content half --no-cpu-baseline
run c1_compare --config c1 --no-cpu-baseline
run c3_compare --config c3 --steps 10 --warmup 3 --no-cpu-baseline
run c4_compare --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e
run c4_hash --config c4 --mode hash --steps 5 --warmup 3 --no-cpu-baseline --no-e2e
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > $O/torchrun1.json 2> $O/torchrun1.err; echo "torchrun rc=$?"
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2_compare.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2_hash2m.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --mode hash --page 2097152 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_detect_compare|k_gather|k_compact_onepass" -s 15 -c 3 -o $O/c2_compare_full $B --no-e2e > $O/n1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_detect_hash_tma|k_compact_onepass" -s 8 -c 2 -o $O/c2_hash2m_full $B --no-e2e --mode hash --page 2097152 > $O/n2.log 2>&1
tail -1 $O/n1.log $O/n2.log
ls -la $O
