# same-box A/B: ring-path metadata through the mapped address (current) vs D2H metadata copies (f8ff49c)
O=gpurun_out/r03v; mkdir -p $O
run() {
  python -c "import __graft_entry__ as g; g.build()"
  for i in 1 2 3; do
    timeout 400 python bench.py --config c2 --dirty 0.1 --no-cpu-baseline --no-e2e > $O/$1_$i.json 2> $O/$1_$i.err
    python -c "import json; d=json.load(open('$O/$1_$i.json')); print('$1', d['value'], d['ms_per_step'], d['step']['frac'], d['step']['link_peak_GBs'], d['parity']['ok'])"
  done
}
run cur
# (the A/B copied the f8ff49c versions of runtime.cu / kernels_image.cu over the tree; files removed since)
# (the A/B copied the f8ff49c versions of runtime.cu / kernels_image.cu over the tree; files removed since)
run pre
