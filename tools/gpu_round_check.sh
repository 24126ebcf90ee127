mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python tools/sanitize_run.py 2>&1 | tail -3
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --target-processes all python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|Error|Hazard|sanitize workload" gpurun_out/sanitize_$tool.log | head -8
done
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -x 2>&1 | tail -4
