mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|sanitize workload" gpurun_out/sanitize_$tool.log | head -3
done
CRUM_HASH_NO_TMA=1 timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_racecheck_notma.log 2>&1
echo "== racecheck (register-staged hash kernel) rc=$?"; grep -E "RACECHECK SUMMARY|sanitize workload" gpurun_out/sanitize_racecheck_notma.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python tools/sanitize_run.py > gpurun_out/sanitize_racecheck_tma.log 2>&1
echo "== racecheck (TMA hash kernel) rc=$?"; grep -E "RACECHECK SUMMARY|sanitize workload" gpurun_out/sanitize_racecheck_tma.log; grep -c "k_detect_hash_tma" gpurun_out/sanitize_racecheck_tma.log; grep "Race reported" gpurun_out/sanitize_racecheck_tma.log | grep -v k_detect_hash_tma | grep -v bulk_g2s | head -3
compute-sanitizer --version | tail -1
