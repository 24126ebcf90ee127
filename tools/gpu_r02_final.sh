# round-2 evidence: smoke, new tests, default line + reference + launch list, config lines, C2 sweep
O=gpurun_out/final; mkdir -p $O $O/sweep
python -c "import __graft_entry__ as g; g.build()"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "mapped" 2>&1 | tail -1
timeout 600 python bench.py > $O/default.json 2> $O/default.err; echo "default rc=$?"
timeout 600 python bench.py --impl reference > $O/reference.json 2> $O/reference.err; echo "reference rc=$?"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
timeout 300 python bench.py --config c1 --steps 200 --warmup 20 > $O/c1.json 2> $O/c1.err; echo "c1 rc=$?"
timeout 600 python bench.py --config c3 --restore-full > $O/c3.json 2> $O/c3.err; echo "c3 rc=$?"
timeout 600 python bench.py --config c4 --mode hash > $O/c4_hash.json 2> $O/c4_hash.err; echo "c4 hash rc=$?"
for c in random half hpgmg; do
  timeout 400 python bench.py --config c2 --compress --content $c --no-cpu-baseline > $O/c2z_$c.json 2> $O/c2z_$c.err; echo "z $c rc=$?"
done
for mode in compare hash; do
for pg in 65536 2097152; do
 for d in 0.0 0.01 0.1 0.5 1.0; do
  f=$O/sweep/c2_${mode}_${pg}_${d}.json
  timeout 600 python bench.py --config c2 --mode $mode --page $pg --dirty $d --no-cpu-baseline > $f 2> ${f%.json}.err
 done
done
done
echo sweep done
