python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python bench.py --config c2 --compress --content random --region-gib 1 --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | grep -v CUDAEvent | grep -E "Invalid|at |by thread|Address|ERROR SUMMARY|Error" | head -30
