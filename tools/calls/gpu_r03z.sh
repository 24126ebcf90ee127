# C1 fine stamps (profiling build), then the round-end sequence on the normal build
bash tools/gpu_r02_c1_stamps.sh > gpurun_out/c1_stamps_fine.txt 2>&1
grep "small stamps" gpurun_out/c1_stamps.txt | tail -13
bash tools/gpu_round_end.sh
