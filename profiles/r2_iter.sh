#!/bin/bash
# Iteration pass: GPU tests, smoke, C3 and C5 bench lines (no CPU baseline).
#   O=<outdir> TESTS=<pytest selection> bash profiles/r2_iter.sh
O=${O:-gpurun_out/iter}
mkdir -p $O
timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -x -q -p no:cacheprovider > $O/gpu_tests.txt 2>&1
tail -5 $O/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
tail -3 $O/smoke.txt
for c in ${CONFIGS:-c3 c5}; do
  timeout 900 python bench.py --config $c --no-cpu-baseline ${BENCH_ARGS} > $O/bench_$c.json 2> $O/bench_$c.err
  tail -c 300 $O/bench_$c.err
  python - $O/bench_$c.json <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print(sys.argv[1], "value", round(d["value"],1), "ms", round(d["ms_per_step"],3), "e2e", round(d["e2e"]["value"],1), "api", round((d.get("e2e_api") or {}).get("value",0),1))
print("clocks", d["clocks"], "roof", {k: d["roofline"].get(k) for k in ("kernel","achieved","frac","frac_of_3xfp16_bound")})
for k,v in sorted(d["roofline"]["classes"].items(), key=lambda kv:-kv[1]["ms_per_step"]): print("  ",k,{a:(round(b,3) if isinstance(b,float) else b) for a,b in v.items()})
PY
done
