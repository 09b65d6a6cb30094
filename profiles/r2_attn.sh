#!/bin/bash
# Per-launch attribution (GR4AD_PROF_DUMP through bench.py's profiled window)
# for C3 and C5, and ncu --set full captures of one C3 Q.X^T and one P.X launch.
O=${O:-gpurun_out/attn}
mkdir -p $O
for c in c3 c5; do
  rm -f $O/dump_$c.tsv
  GR4AD_PROF_DUMP=$O/dump_$c.tsv timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 > $O/bench_$c.json 2> $O/bench_$c.err
  python profiles/launch_summary.py $O/dump_$c.tsv > $O/launches_$c.txt
  head -40 $O/launches_$c.txt
done
GR4AD_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-graph --no-cpu-baseline \
  > /dev/null 2> $O/trace_c3.txt
python - $O/trace_c3.txt > $O/attn_idx.txt <<'PY'
import sys
lines=[l for l in open(sys.argv[1]) if l.startswith("gemm_tc ")]
qk=[i for i,l in enumerate(lines) if " mode=1 " in l and "M=512" in l]
pv=[i for i,l in enumerate(lines) if " mode=2 " in l and "M=512" in l]
print(qk[0], pv[0], len(lines))
PY
cat $O/attn_idx.txt
read QK PV N < $O/attn_idx.txt
B="python bench.py --steps 1 --warmup 1 --no-graph --no-cpu-baseline"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc \
  -s $QK -c 1 -o $O/prof_qk_c3 $B > $O/ncu_qk.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc \
  -s $PV -c 1 -o $O/prof_pv_c3 $B > $O/ncu_pv.log 2>&1
ls -la $O
