#!/bin/bash
# C4 sweep with concurrent serving threads (serve_batch from 1 / 2 / 3 workers)
O=${O:-gpurun_out/wk}
mkdir -p $O
for w in 1 2 3; do
  timeout 900 python serving_bench.py --model c5 --duration 2 --workers $w > $O/serving_c5_w$w.jsonl 2> $O/serving_c5_w$w.err
  python - $O/serving_c5_w$w.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    d=json.loads(l)
    if "capacity_req_s" in d: print(d["model"], "workers", d["workers"], "capacity", round(d["capacity_req_s"])); continue
    print("  load", d["offered_load"], "ach", round(d["achieved_req_s"]), "w", d["last_level_width"]["median"], "p50", round(d["latency_ms"]["p50"],1), "p99", round(d["latency_ms"]["p99"],1))
PY
  tail -2 $O/serving_c5_w$w.err
done
