#!/bin/bash
# Profile captures for the round (run under gpurun on 1 GPU; writes gpurun_out/prof_*).
set -x
O=gpurun_out
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file $O/prof_launches_c2.csv python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 268 -c 261 --csv \
  --log-file $O/prof_launches_c3.csv python bench.py --config c3 --steps 1 --warmup 3 --no-graph --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 40 -c 2 \
  -o $O/prof_gemm_tc_c3 python bench.py --config c3 --steps 1 --warmup 3 --no-graph --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:topk_select -s 3 -c 1 \
  -o $O/prof_topk_c3 python bench.py --config c3 --steps 1 --warmup 3 --no-graph --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:fused_small -s 3 -c 1 \
  -o $O/prof_fused_c2 python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline > /dev/null 2>&1
ls -la $O
