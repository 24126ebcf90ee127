# ncu --set full of one k_zenc launch on HPGMG-like content (C2 compressed)
O=gpurun_out/r04i; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_zenc --launch-skip 20 -c 1 -o $O/zenc_hpgmg python tools/trace_e2e.py 65536 0.1 --compress --content hpgmg > $O/ncu.log 2>&1; echo "ncu rc=$?"
