#!/bin/bash
# (the GR4AD_PDL switch was removed with the experiment; kept as the record of the A/B)
# A/B: programmatic dependent launch of the GEMMs (GR4AD_PDL=0 / 1), bench lines
O=${O:-gpurun_out/pdl}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_big.py tests/test_gpu_api.py -x -q -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do
  for p in 0 1; do
    for c in c5 c3; do
      GR4AD_PDL=$p timeout 900 python bench.py --config $c --no-cpu-baseline > $O/b_${c}_$p.json 2> /dev/null
      python -c "import json;d=json.load(open('$O/b_${c}_$p.json'));print('$c pdl=$p', round(d['ms_per_step'],3), 'clk', d['clocks']['sm_mhz'], 'e2e', round(d['e2e']['value']))"
    done
  done
done
