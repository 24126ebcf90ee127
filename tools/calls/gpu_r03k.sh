# small path: distributed metadata writes + parallel header CRC: parity, C1 lines, phase stamps
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r03k; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_edges.py -q -k "small or every_path or edge or c1 or gather" 2>&1 | tail -2
timeout 300 python bench.py --config c1 --steps 200 --warmup 20 --no-cpu-baseline > $O/c1.json 2> $O/c1.err; echo "c1 rc=$?"
python -c "import json; d=json.load(open('$O/c1.json')); print(d['value'], d['ms_per_step'], d['call_latency'], d['parity']['ok'])"
python -c "
import sys; sys.path.insert(0,'paper_1808_00117_b200'); import build; build.build(force=True, extra=['-DCRUM_SMALL_STAMPS'])"
timeout 300 python tools/c1_latency.py > $O/c1_stamps.txt 2>&1
grep "small stamps" $O/c1_stamps.txt | tail -24 | sort | uniq -c | sort -k4 | head -30
python paper_1808_00117_b200/build.py --force > /dev/null
