#!/bin/bash
# Round 2 first GPU pass: tests (incl. the bench-shaped C3/C5/C4 parity),
# smoke, the default (C3) bench line, and ncu captures of the C3 attention
# products (Q.K^T vs P.V) located through GR4AD_TRACE.
O=gpurun_out/r2a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gpu_tests.txt 2>&1
tail -3 $O/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
tail -3 $O/smoke.txt
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
tail -c 600 $O/bench_c3.json
GR4AD_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-graph --no-cpu-baseline \
  > /dev/null 2> $O/trace_c3.txt
python - $O/trace_c3.txt > $O/attn_idx.txt <<'PY'
import sys
lines=[l for l in open(sys.argv[1]) if l.startswith("gemm_tc ")]
# one decode per BeamDecoder.run; the first run is the launch count probe
n=len(lines)
qk=[i for i,l in enumerate(lines) if " mode=1 " in l and "M=512" in l]
pv=[i for i,l in enumerate(lines) if " mode=2 " in l and "M=512" in l]
print(qk[0], pv[0], n)
PY
cat $O/attn_idx.txt
read QK PV N < $O/attn_idx.txt
B="python bench.py --steps 1 --warmup 1 --no-graph --no-cpu-baseline"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc \
  -s $QK -c 1 -o $O/prof_qk_c3 $B > $O/ncu_qk.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc \
  -s $PV -c 1 -o $O/prof_pv_c3 $B > $O/ncu_pv.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout -s KILL 900 ncu --metrics $M --clock-control none -c 1200 --csv \
  --log-file $O/launches_c3.csv $B > /dev/null 2>&1
ls -la $O
