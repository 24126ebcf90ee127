mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01b_launches_c2_compare.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01b_launches_c2_hash64k.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --mode hash > /dev/null 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01b_launches_c2_zhalf.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --compress --content half > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_detect_compare|k_gather" -s 10 -c 2 -o gpurun_out/r01b_c2_compare $B --no-e2e > gpurun_out/n1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_detect_hash_tma" -s 4 -c 1 -o gpurun_out/r01b_c2_hash64k_tma $B --no-e2e --mode hash > gpurun_out/n2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_detect_hash_tma" -s 4 -c 1 -o gpurun_out/r01b_c2_hash2m_tma $B --no-e2e --mode hash --page 2097152 > gpurun_out/n3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_zsize|k_zwrite|k_zdecode" -s 6 -c 3 -o gpurun_out/r01b_c2_zhalf $B --compress --content half > gpurun_out/n4.log 2>&1
tail -1 gpurun_out/n1.log gpurun_out/n2.log gpurun_out/n3.log gpurun_out/n4.log
ls -la gpurun_out
