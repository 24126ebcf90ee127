# mapped-store range pipeline (small payloads): parity, traces, C2 sweep lines; encoder launch times
mkdir -p gpurun_out/r03b
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for d in 0.0 0.01; do timeout 300 python tools/trace_e2e.py 65536 $d > gpurun_out/r03b/trace_$d.txt 2>&1; done
for d in 0.0 0.01 0.1; do
  timeout 400 python bench.py --config c2 --dirty $d --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r03b/c2_$d.json 2> gpurun_out/r03b/c2_$d.err; echo "c2 $d rc=$?"
done
timeout 400 python bench.py --config c2 --mode hash --page 2097152 --dirty 0.0 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r03b/c2_hash2m_0.0.json 2> gpurun_out/r03b/c2_hash2m_0.0.err
timeout 400 python bench.py --config c2 --mode hash --page 2097152 --dirty 0.1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r03b/c2_hash2m_0.1.json 2> gpurun_out/r03b/c2_hash2m_0.1.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_z --csv --log-file gpurun_out/r03b/zenc_launches.csv python tools/trace_e2e.py 65536 0.1 --compress > /dev/null 2>&1; echo "ncu rc=$?"
