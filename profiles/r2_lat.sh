#!/bin/bash
# Iteration on the fused latent block: GPU tests, smoke, C3 / C5 lines, and
# ncu --set full of the two latent-block kernels (text pages only).
O=${O:-gpurun_out/lat}
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
print(sys.argv[1], "value", round(d["value"],1), "ms", round(d["ms_per_step"],3), "e2e", round(d["e2e"]["value"],1), "clk", d["clocks"]["sm_mhz"])
for k,v in sorted(d["roofline"]["classes"].items(), key=lambda kv:-kv[1]["ms_per_step"]): print("  ",k,{a:(round(b,3) if isinstance(b,float) else b) for a,b in v.items()})
PY
done
B="python bench.py --steps 1 --warmup 1 --no-graph --no-cpu-baseline"
NF="ncu --set full --clock-control none --import-source on"
timeout -s KILL 600 $NF -k regex:latent_attn -s 8 -c 1 -o $O/prof_x $B > $O/ncu_x.log 2>&1
timeout -s KILL 600 $NF -k regex:latent_out -s 8 -c 1 -o $O/prof_y $B > $O/ncu_y.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout -s KILL 900 ncu --metrics $M --clock-control none -c 1500 --csv \
  --log-file $O/launches_c3.csv $B > /dev/null 2>&1
for r in $O/*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv > $b.source.csv 2>/dev/null
  gzip -f $b.source.csv
  rm -f $r
done
du -sh $O
