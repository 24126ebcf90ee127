# Session evidence after the page-group hash kernel, the compaction fill and
# the in-run parity check: sanitizers, full GPU suite, smoke, bench lines for
# every configuration, reference arm, launch lists, ncu --set full captures.
O=gpurun_out/r01d
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --target-processes all python tools/sanitize_run.py > $O/sanitize_$tool.txt 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|sanitize workload" $O/sanitize_$tool.txt | head -3
done
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -2
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
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "crum_checkpoint_gather_device/" -k regex:"k_detect_compare|k_gather|k_compact_onepass" -s 3 -c 3 -o $O/c2_compare_full $B --no-e2e > $O/n1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_detect_hash_pair|k_compact_onepass" -s 8 -c 2 -o $O/c2_hash2m_full $B --no-e2e --mode hash --page 2097152 > $O/n2.log 2>&1
tail -1 $O/n1.log $O/n2.log
ls $O
