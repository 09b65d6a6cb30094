#!/bin/bash
# GPU tests + smoke + default bench line.  O=<outdir> (default gpurun_out/r2c)
O=${O:-gpurun_out/r2c}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${PYTEST_ARGS} > $O/gpu_tests.txt 2>&1
tail -5 $O/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
tail -3 $O/smoke.txt
timeout 900 python bench.py ${BENCH_ARGS} > $O/bench.json 2> $O/bench.err
tail -c 300 $O/bench.err
python - $O/bench.json <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], "api", d.get("e2e_api"))
print("clocks", d["clocks"], "roof", {k: d["roofline"][k] for k in ("kernel","achieved","frac")})
for k,v in sorted(d["roofline"]["classes"].items(), key=lambda kv:-kv[1]["ms_per_step"]): print("  ",k,v)
PY
