mkdir -p gpurun_out/sanitizer
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python tools/sanitize_run.py 2>&1 | tail -2
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --target-processes all python tools/sanitize_run.py > gpurun_out/sanitizer/r02_$tool.txt 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|Error|Hazard|sanitize workload" gpurun_out/sanitizer/r02_$tool.txt | head -8
done
