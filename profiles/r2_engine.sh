#!/bin/bash
# Engine pass: GPU API tests, C4 sweep through ServingEngine (batch-level
# load widths, bucket-padded batches), cProfile of the engine at two loads.
O=${O:-gpurun_out/eng}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_api.py -x -q -p no:cacheprovider > $O/gpu_api.txt 2>&1
tail -3 $O/gpu_api.txt
timeout 900 python serving_bench.py --model c5 --duration 2 > $O/serving_c5.jsonl 2> $O/serving_c5.err
cat $O/serving_c5.jsonl; tail -5 $O/serving_c5.err
timeout 600 python serving_bench.py --model c5 --duration 2 --loads 0.5 --profile > $O/prof_c5.jsonl 2> $O/prof_c5.err
cat $O/prof_c5.jsonl; head -80 $O/prof_c5.err
timeout 600 python bench.py --config c5 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
python -c "import json;d=json.load(open('$O/bench_c5.json'));print('c5', d['value'], d['ms_per_step'], 'api', d['e2e_api']['value'], d['e2e_api']['ms_per_step'], d['e2e_api']['host_materialize_ms'])"
