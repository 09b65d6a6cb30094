#!/bin/bash
# Round-2 final evidence pass (1 GPU): GPU tests + smoke, bench lines (C3
# default with CPU baseline, reference arm, C1 / C2 / C5), the C4 serving
# sweeps through ServingEngine, launch lists (C3, C5, C2) and ncu --set full
# of the top kernels (text pages only).
O=${O:-gpurun_out/final}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.txt 2>&1
tail -3 $O/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
tail -2 $O/smoke.txt
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --impl reference > $O/bench_reference_c3.json 2> $O/bench_ref.err
for c in c5 c2 c1; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
for f in $O/bench_*.json; do echo $f; python - $f <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
if d.get("impl")=="reference": print("  ref", d["value"], d.get("cpu_baseline")); raise SystemExit
print("  value", round(d["value"],1), "ms", round(d["ms_per_step"],3), "e2e", round(d["e2e"]["value"],1), "api", round(d.get("e2e_api",{}).get("value",0),1), "clk", d["clocks"]["sm_mhz"], d["clocks"].get("reasons"))
print("  roofline", {k:v for k,v in d["roofline"].items() if k!="classes"})
PY
done
timeout 900 python serving_bench.py --model c5 --duration 2 > $O/serving_c4_c5model.jsonl 2> $O/serving_c5.err
timeout 600 python serving_bench.py --model c2 --duration 2 > $O/serving_c4_c2model.jsonl 2> $O/serving_c2.err
cut -c1-400 $O/serving_c4_c5model.jsonl
B="python bench.py --steps 1 --warmup 1 --no-graph --no-cpu-baseline"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout -s KILL 900 ncu --metrics $M --clock-control none -c 1500 --csv --log-file $O/launches_c3.csv $B > /dev/null 2>&1
timeout -s KILL 900 ncu --metrics $M --clock-control none -c 1500 --csv --log-file $O/launches_c5.csv $B --config c5 > /dev/null 2>&1
timeout -s KILL 300 ncu --metrics $M --clock-control none -c 400 --csv --log-file $O/launches_c2.csv $B --config c2 > /dev/null 2>&1
GR4AD_TRACE=1 timeout 300 $B > /dev/null 2> $O/trace_c3.txt
python - $O/trace_c3.txt > $O/idx.txt <<'PY'
import sys
lines=[l for l in open(sys.argv[1]) if l.startswith("gemm_tc ")]
def first(*keys):
    return next((i for i,l in enumerate(lines) if all(k in l for k in keys)), 0)
print(first("M=131072 ", "N=2048 ", "K=1024 "), first("M=131072 ", "N=4096 "),
      first("M=131072 ", "N=1024 ", "K=2048 "), first("M=768 ", "N=2048 ", "K=1024 "))
PY
read W1 LG W2 TW1 < $O/idx.txt
echo "idx $W1 $LG $W2 $TW1"
NF="ncu --set full --clock-control none --import-source on"
timeout -s KILL 600 $NF -k regex:gemm_tc -s $W1 -c 1 -o $O/prof_gemm_w1 $B > $O/ncu1.log 2>&1
timeout -s KILL 600 $NF -k regex:gemm_tc -s $LG -c 1 -o $O/prof_gemm_logits $B > $O/ncu2.log 2>&1
timeout -s KILL 600 $NF -k regex:gemm_tc -s $W2 -c 1 -o $O/prof_gemm_w2 $B > $O/ncu3.log 2>&1
timeout -s KILL 600 $NF -k regex:gemm_tc -s $TW1 -c 1 -o $O/prof_gemm_trunk_w1 $B > $O/ncu4.log 2>&1
timeout -s KILL 600 $NF -k regex:topk_select -s 1 -c 1 -o $O/prof_topk $B > $O/ncu5.log 2>&1
timeout -s KILL 600 $NF -k regex:topk_select -s 0 -c 1 -o $O/prof_topk_l0 $B > $O/ncu6.log 2>&1
timeout -s KILL 600 $NF -k regex:self_attn -s 23 -c 1 -o $O/prof_self $B > $O/ncu7.log 2>&1
timeout -s KILL 600 $NF -k regex:latent_attn -s 8 -c 1 -o $O/prof_lat_x $B > $O/ncu8.log 2>&1
timeout -s KILL 600 $NF -k regex:latent_out -s 8 -c 1 -o $O/prof_lat_y $B > $O/ncu9.log 2>&1
timeout -s KILL 600 $NF -k regex:ln_rows_split -s 8 -c 1 -o $O/prof_ln3 $B > $O/ncu10.log 2>&1
timeout -s KILL 300 $NF -k regex:fused_mma -s 1 -c 1 -o $O/prof_fused_c2 $B --config c2 > $O/ncu11.log 2>&1
for r in $O/*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv > $b.source.csv 2>/dev/null
  gzip -f $b.source.csv
  rm -f $r
done
python profiles/ncu_digest.py $O/prof_*.raw.csv > $O/ncu_summary.txt
cat $O/ncu_summary.txt | head -40
rm -f $O/trace_c3.txt
du -sh $O
