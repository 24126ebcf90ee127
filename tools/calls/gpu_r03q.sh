# compressed gathers: range lookahead A/B (2 shipped / 1 / all), C2 random / half / hpgmg
O=gpurun_out/r03q; mkdir -p $O
run() {
  python -c "import __graft_entry__ as g; g.build()"
  for c in random half hpgmg; do
    timeout 400 python bench.py --config c2 --compress --content $c --no-cpu-baseline --no-e2e > $O/la${LA}_$c.json 2> $O/la${LA}_$c.err
    python -c "import json; d=json.load(open('$O/la${LA}_$c.json')); print('la$LA $c', d['value'], d['ms_per_step'], d['parity']['ok'])"
  done
  timeout 300 python tools/trace_e2e.py 65536 0.1 --compress > $O/la${LA}_trace_random.txt 2>&1
}
LA=2 run
python - <<'PY'
p='paper_1808_00117_b200/csrc/runtime.cu'; s=open(p).read()
a=s.index("int gather_z("); b=s.index("\n}\n", a)
f=s[a:b]
f=f.replace("while (enq < nr && enq < 2)","while (enq < nr && enq < 1)").replace("while (enq < nr && enq <= ci + 2)","while (enq < nr && enq <= ci + 1)")
open(p,'w').write(s[:a]+f+s[b:])
PY
LA=1 run
python - <<'PY'
p='paper_1808_00117_b200/csrc/runtime.cu'; s=open(p).read()
a=s.index("int gather_z("); b=s.index("\n}\n", a)
f=s[a:b]
f=f.replace("while (enq < nr && enq < 1)","while (enq < nr && enq < 64)").replace("while (enq < nr && enq <= ci + 1)","while (enq < nr && enq <= ci + 64)")
open(p,'w').write(s[:a]+f+s[b:])
PY
LA=all run
