#!/bin/bash
# A/B on one box: alternate the committed build (profiles/libgr4ad_base.so)
# and the working tree's build, R rounds, config $1 (default c3).
C=${1:-c3}; R=${2:-3}
for i in $(seq $R); do
  for v in base new; do
    if [ $v = base ]; then export GR4AD_LIB=profiles/libgr4ad_base.so; else unset GR4AD_LIB; fi
    echo -n "$v "; bash profiles/bench_lines.sh $C
  done
done
