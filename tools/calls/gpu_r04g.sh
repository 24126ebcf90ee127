# ring pipeline over the halving ranges for 16-64 MiB previous payloads: parity + C2 lines at 2 / 3 / 5 %
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -q -k "mapped or every_path or gather or deferred or capacity or full_size" 2>&1 | tail -1
O=gpurun_out/r04g; mkdir -p $O
for cfg in "compare 2097152" "hash 65536" "hash 2097152"; do set -- $cfg
  for d in 0.02 0.03 0.05; do
  f=$O/c2_$1_$2_$d.json
  timeout 600 python bench.py --config c2 --mode $1 --page $2 --dirty $d --no-cpu-baseline --no-e2e > $f 2> ${f%.json}.err
  python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$1 $2 $d', 'value', d['value'], 'ms', d['ms_per_step'], 'step frac', d['step']['frac'], 'parity', d['parity']['ok'])"
  done
done
