#!/bin/bash
# Iteration: GPU tests, smoke, C3 / C5 lines, C4 through ServingEngine,
# launch lists (C3, C5) after the selection / latent-tile / derived-weight changes.
O=${O:-gpurun_out/it3}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gpu_tests.txt 2>&1
tail -15 $O/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
tail -3 $O/smoke.txt
for c in c3 c5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  tail -c 300 $O/bench_$c.err
  python - $O/bench_$c.json <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print(sys.argv[1], "value", round(d["value"],1), "ms", round(d["ms_per_step"],3), "e2e", round(d["e2e"]["value"],1), "api", round(d["e2e_api"]["value"],1), "clk", d["clocks"]["sm_mhz"])
for k,v in sorted(d["roofline"]["classes"].items(), key=lambda kv:-kv[1]["ms_per_step"]): print("  ",k,{a:(round(b,3) if isinstance(b,float) else b) for a,b in v.items()})
PY
done
timeout 900 python serving_bench.py --model c5 --duration 2 > $O/serving_c4_c5model.jsonl 2> $O/serving_c5.err
tail -12 $O/serving_c4_c5model.jsonl; tail -5 $O/serving_c5.err
B="python bench.py --steps 1 --warmup 1 --no-graph --no-cpu-baseline"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout -s KILL 900 ncu --metrics $M --clock-control none -c 1500 --csv \
  --log-file $O/launches_c3.csv $B > /dev/null 2>&1
timeout -s KILL 900 ncu --metrics $M --clock-control none -c 1500 --csv \
  --log-file $O/launches_c5.csv $B --config c5 > /dev/null 2>&1
du -sh $O
