#!/bin/bash
# (split-K experiment record: the GR4AD_KSPLIT / GR4AD_SMALLM switches were removed with it)
# ncu of the trunk's first W1 product (M=768, epi 10) under split-K variants
O=${O:-gpurun_out/ksn}
mkdir -p $O
B="python bench.py --config c5 --steps 1 --warmup 1 --no-graph --no-cpu-baseline"
NF="ncu --set full --clock-control none --import-source on"
for v in "KS=2" "KS=4" "KS=8"; do
  case $v in KS=*) export GR4AD_KSPLIT=${v#KS=}; unset GR4AD_SMALLM;; SM=1) export GR4AD_KSPLIT=4 GR4AD_SMALLM=1;; esac
  timeout -s KILL 600 $NF -k regex:gemm_tc -s 2 -c 1 -o $O/v_${v/=/} $B > $O/ncu_${v/=/}.log 2>&1
done
for r in $O/*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page source --csv > $b.source.csv 2>/dev/null
  gzip -f $b.source.csv
  rm -f $r
done
python profiles/ncu_digest.py $O/v_*.raw.csv
