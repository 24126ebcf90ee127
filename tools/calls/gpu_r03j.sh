# C1 phase stamps (profiling build, -DCRUM_SMALL_STAMPS), then the normal build back
python -c "
import sys; sys.path.insert(0,'paper_1808_00117_b200'); import build; build.build(force=True, extra=['-DCRUM_SMALL_STAMPS'])"
timeout 300 python tools/c1_latency.py > gpurun_out/c1_stamps.txt 2>&1
grep "small stamps" gpurun_out/c1_stamps.txt | tail -32 | sort | uniq -c | sort -rn | head -40
python paper_1808_00117_b200/build.py --force > /dev/null
