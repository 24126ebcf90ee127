# host pipeline range cap A/B: F/8 (shipped) vs F/4 vs F/2 on C2 compare / hash 64 KiB at 10 %, C4 compare
O=gpurun_out/r03o; mkdir -p $O
run() {
  python -c "import __graft_entry__ as g; g.build()"
  for cfg in "compare 65536" "hash 2097152"; do set -- $cfg
    timeout 400 python bench.py --config c2 --mode $1 --page $2 --dirty 0.1 --no-cpu-baseline > $O/cap${CAP}_c2_$1.json 2> $O/cap${CAP}_c2_$1.err
    python -c "import json; d=json.load(open('$O/cap${CAP}_c2_$1.json')); print('cap$CAP c2 $1', d['value'], d['ms_per_step'], d['step']['frac'], d['parity']['ok'])"
  done
  timeout 600 python bench.py --no-cpu-baseline > $O/cap${CAP}_c4.json 2> $O/cap${CAP}_c4.err
  python -c "import json; d=json.load(open('$O/cap${CAP}_c4.json')); print('cap$CAP c4', d['value'], d['ms_per_step'], d['step']['frac'], d['parity']['ok'])"
  timeout 300 python tools/trace_e2e.py 65536 0.1 > $O/cap${CAP}_trace.txt 2>&1
}
CAP=8 run
for v in 4 2; do
  sed -i "s|const uint64_t target_max = std::max(kMinRangeBytes, F / [0-9]*);|const uint64_t target_max = std::max(kMinRangeBytes, F / $v);|" paper_1808_00117_b200/csrc/runtime.cu
  CAP=$v run
done
