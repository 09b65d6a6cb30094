#!/bin/bash
# Round evidence (1 GPU, under gpurun): bench lines, reference arm, serving
# sweep, ncu launch lists and --set full captures, fused-kernel phase stamps.
#   gpurun --timeout 2400 -- bash profiles/run_round.sh
# Outputs land in gpurun_out/round/; copy the summaries into profiles/<round>/.
O=gpurun_out/round
mkdir -p $O
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --impl reference > $O/bench_reference_c2.json 2> $O/bench_ref.err
timeout 300 python bench.py --config c1 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c5 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python serving_bench.py --model c5 > $O/serving_c4_c5model.jsonl 2> $O/serving_c5.err
timeout 300 python serving_bench.py --model c2 > $O/serving_c4_c2model.jsonl 2> $O/serving_c2.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
B="python bench.py --steps 1 --warmup 1 --no-graph --no-cpu-baseline"
timeout -s KILL 300 ncu --metrics $M --clock-control none -c 400 --csv \
  --log-file $O/launches_c2.csv $B > /dev/null 2>&1
timeout -s KILL 900 ncu --metrics $M --clock-control none -c 1200 --csv \
  --log-file $O/launches_c3.csv $B --config c3 > /dev/null 2>&1
timeout -s KILL 900 ncu --metrics $M --clock-control none -c 1200 --csv \
  --log-file $O/launches_c5.csv $B --config c5 > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:fused_mma \
  -s 1 -c 1 -o $O/prof_fused_c2 $B > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc \
  -s 100 -c 6 -o $O/prof_gemm_tc_c3 $B --config c3 > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:topk_select \
  -s 2 -c 1 -o $O/prof_topk_c3 $B --config c3 > /dev/null 2>&1
if [ -f profiles/libgr4ad_timing.so ]; then
  GR4AD_LIB=profiles/libgr4ad_timing.so timeout 300 python profiles/fused_phases.py --batch 296 \
    > $O/fused_phases_c2.txt 2>&1
fi
timeout 120 python profiles/h2d_probe.py > $O/h2d.txt 2>&1
ls -la $O
