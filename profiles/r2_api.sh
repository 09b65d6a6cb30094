#!/bin/bash
# API / engine iteration: GPU API tests, C3 / C5 / C2 bench lines (api e2e),
# C4 sweeps through ServingEngine (C5 and C2 models).
O=${O:-gpurun_out/api}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider > $O/gpu_api.txt 2>&1
tail -3 $O/gpu_api.txt
for c in c5 c3 c2; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  python -c "import json;d=json.load(open('$O/bench_$c.json'));a=d['e2e_api'];print('$c', round(d['value'],1), d['ms_per_step'], 'api', round(a['value'],1), round(a['ms_per_step'],2), 'mat', round(a['host_materialize_ms'],2))"
done
timeout 900 python serving_bench.py --model c5 --duration 2 > $O/serving_c5.jsonl 2> $O/serving_c5.err
timeout 600 python serving_bench.py --model c2 --duration 2 > $O/serving_c2.jsonl 2> $O/serving_c2.err
for m in c5 c2; do python - $O/serving_$m.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    d=json.loads(l)
    if "capacity_req_s" in d: print(d["model"], "capacity", round(d["capacity_req_s"])); continue
    print("  load", d["offered_load"], "ach", round(d["achieved_req_s"]), "w", d["last_level_width"]["median"], "p50", round(d["latency_ms"]["p50"],1), "p99", round(d["latency_ms"]["p99"],1))
PY
done
tail -3 $O/serving_c2.err
