#!/bin/bash
# Profile captures for the round (run under gpurun on 1 GPU; writes gpurun_out/prof_*).
# Launch lists: every launch of `bench.py --steps 1 --warmup 1 --no-graph` (warm-up step included;
# per-launch times are cold-cache and serialised -- shares, not absolutes, compare with bench.py).
set -x
O=gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-graph --no-cpu-baseline"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout -s KILL 300 ncu --metrics $M --clock-control none -c 400 --csv \
  --log-file $O/prof_launches_c2.csv $B > /dev/null 2>&1
timeout -s KILL 900 ncu --metrics $M --clock-control none -c 1200 --csv \
  --log-file $O/prof_launches_c3.csv $B --config c3 > /dev/null 2>&1
# full sections: the level-2 GEMMs of C3 (largest launches), window top-k, fused C2 decode
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc \
  -s 100 -c 6 -o $O/prof_gemm_tc_c3 $B --config c3 > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:topk_select \
  -s 2 -c 1 -o $O/prof_topk_c3 $B --config c3 > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:fused_mma \
  -s 1 -c 1 -o $O/prof_fused_c2 $B > /dev/null 2>&1
ls -la $O
