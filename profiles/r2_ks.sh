#!/bin/bash
# GPU tests, then per-launch attribution (GR4AD_PROF_DUMP) of C3 / C5 steps
O=${O:-gpurun_out/ks}
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gpu_tests.txt 2>&1
tail -3 $O/gpu_tests.txt
for c in c3 c5; do
  rm -f $O/dump_$c.txt
  GR4AD_PROF_DUMP=$O/dump_$c.txt timeout 900 python bench.py --config $c --no-cpu-baseline --steps 3 > $O/b_$c.json 2> $O/b_$c.err
  tail -c 200 $O/b_$c.err
  python profiles/launch_summary.py $O/dump_$c.txt > $O/summary_$c.txt
  head -1 $O/summary_$c.txt; grep "M=768\|M=256 " $O/summary_$c.txt
done
