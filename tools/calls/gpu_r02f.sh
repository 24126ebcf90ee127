mkdir -p gpurun_out/r02f
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "crum_checkpoint_gather/" -c 60 --csv --log-file gpurun_out/r02f/launches_z_hpgmg.csv python bench.py --config c2 --compress --content hpgmg --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_zenc -s 2 -c 1 -o gpurun_out/r02f/zenc_hpgmg python bench.py --config c2 --compress --content hpgmg --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu2 rc=$?"
ls -la gpurun_out/r02f
