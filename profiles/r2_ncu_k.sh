#!/bin/bash
# ncu --set full of one launch of kernel regex $K (skip $SKIP of them) at config $C
O=${O:-gpurun_out/ncuk}
mkdir -p $O
B="python bench.py --steps 1 --warmup 1 --no-graph --no-cpu-baseline --config ${C:-c3}"
for k in $K; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$k \
    -s ${SKIP:-2} -c 1 -o $O/prof_$k $B > $O/ncu_$k.log 2>&1
  tail -3 $O/ncu_$k.log
done
ls -la $O
