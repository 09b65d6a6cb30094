#!/bin/bash
# Round 2, second GPU pass on the factored / latent-attention path: GPU tests,
# smoke, the default (C3) bench line with its CPU baseline, C5, the C3 launch
# list, and ncu --set full captures of the top kernels (trace-located).
O=${O:-gpurun_out/r2b}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gpu_tests.txt 2>&1
  tail -15 $O/gpu_tests.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
  tail -3 $O/smoke.txt
fi
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
tail -c 400 $O/bench_c3.json; echo
timeout 600 python bench.py --config c5 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
tail -c 200 $O/bench_c5.json; echo
B="python bench.py --steps 1 --warmup 1 --no-graph --no-cpu-baseline"
GR4AD_TRACE=1 timeout 300 $B > /dev/null 2> $O/trace_c3.txt
python - $O/trace_c3.txt > $O/idx.txt <<'PY'
import sys
lines=[l for l in open(sys.argv[1]) if l.startswith("gemm_tc ")]
def first(*keys):
    return next(i for i,l in enumerate(lines) if all(k in l for k in keys))
print(first("M=131072 ", "N=2048 ", "K=1024 "), first("M=131072 ", "N=1024 ", "K=16 "),
      first("M=131072 ", "N=4096 "))
PY
cat $O/idx.txt
read W1 KV LG < $O/idx.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout -s KILL 900 ncu --metrics $M --clock-control none -c 1500 --csv \
  --log-file $O/launches_c3.csv $B > /dev/null 2>&1
NF="ncu --set full --clock-control none --import-source on"
timeout -s KILL 600 $NF -k regex:gemm_tc -s $W1 -c 1 -o $O/prof_gemm_w1 $B > $O/ncu1.log 2>&1
timeout -s KILL 600 $NF -k regex:gemm_tc -s $KV -c 1 -o $O/prof_gemm_k16 $B > $O/ncu2.log 2>&1
timeout -s KILL 600 $NF -k regex:gemm_tc -s $LG -c 1 -o $O/prof_gemm_logits $B > $O/ncu3.log 2>&1
timeout -s KILL 600 $NF -k regex:latent_attn -s 8 -c 1 -o $O/prof_latent $B > $O/ncu4.log 2>&1
timeout -s KILL 600 $NF -k regex:ln_rows_split -s 24 -c 1 -o $O/prof_ln $B > $O/ncu5.log 2>&1
timeout -s KILL 600 $NF -k regex:topk_select -s 1 -c 1 -o $O/prof_topk $B > $O/ncu6.log 2>&1
timeout -s KILL 600 $NF -k regex:self_attn -s 20 -c 1 -o $O/prof_self $B > $O/ncu7.log 2>&1
# keep what travels back small: text pages of every capture, no .ncu-rep
for r in $O/*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv > $b.source.csv 2>/dev/null
  gzip -f $b.source.csv
  rm -f $r
done
rm -f $O/trace_c3.txt
du -sh $O; ls -la $O
