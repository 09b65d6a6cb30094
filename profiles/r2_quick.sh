#!/bin/bash
# Quick iteration: GPU parity tests + C3 / C5 bench lines (class breakdown).
O=${O:-gpurun_out/q}
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${TESTS:-} > $O/gpu_tests.txt 2>&1
tail -3 $O/gpu_tests.txt
for c in ${CONFIGS:-c3 c5}; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  tail -c 300 $O/bench_$c.err
  python - $O/bench_$c.json <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print(sys.argv[1], "value", round(d["value"],1), "ms", round(d["ms_per_step"],3), "e2e", round(d["e2e"]["value"],1), "api", round(d["e2e_api"]["value"],1), "clk", d["clocks"]["sm_mhz"])
for k,v in sorted(d["roofline"]["classes"].items(), key=lambda kv:-kv[1]["ms_per_step"]): print("  ",k,{a:(round(b,3) if isinstance(b,float) else b) for a,b in v.items()})
PY
done
