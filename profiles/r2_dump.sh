#!/bin/bash
# Per-launch attribution through bench.py's profiled window (GR4AD_PROF_DUMP).
O=${O:-gpurun_out/dump}
mkdir -p $O
for c in ${CONFIGS:-c3 c5}; do
  rm -f $O/dump_$c.tsv
  GR4AD_PROF_DUMP=$O/dump_$c.tsv timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 > $O/bench_$c.json 2> $O/bench_$c.err
  python profiles/launch_summary.py $O/dump_$c.tsv > $O/launches_$c.txt
  head -${TOP:-30} $O/launches_$c.txt
done
