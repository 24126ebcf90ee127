# end-of-round C2 sweep (0 / 1 / 2 / 10 / 50 / 100 %, 64 KiB and 2 MiB pages, compare and hash) + default line
O=gpurun_out/sweep_end; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python bench.py > $O/default.json 2> $O/default.err; echo "default rc=$?"
for mode in compare hash; do
for pg in 65536 2097152; do
 for d in 0.0 0.01 0.02 0.1 0.5 1.0; do
  f=$O/c2_${mode}_${pg}_${d}.json
  timeout 600 python bench.py --config c2 --mode $mode --page $pg --dirty $d --no-cpu-baseline > $f 2> ${f%.json}.err
 done
done
done
echo sweep done
