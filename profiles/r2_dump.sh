#!/bin/bash
# Per-launch live attribution (GR4AD_PROF_DUMP) of the C3 and C5 bench steps.
O=${O:-gpurun_out/dump}
mkdir -p $O
for c in c3 c5; do
  rm -f $O/dump_$c.txt
  GR4AD_PROF_DUMP=$O/dump_$c.txt timeout 900 python bench.py --config $c --no-cpu-baseline --steps 3 > $O/b_$c.json 2> $O/b_$c.err
  python profiles/launch_summary.py $O/dump_$c.txt > $O/summary_$c.txt
  head -45 $O/summary_$c.txt
done
