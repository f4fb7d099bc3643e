#!/bin/bash
# A/B: group sync path host scatter (base) vs scatter kernel + wait (prev), cfg 3 with 400K-key tables
tag=${1:-r02ak}
out=gpurun_out/$tag; mkdir -p $out
for i in 1 2; do
  timeout 900 python tools/bench_cfg3.py --keys-per-table 400000 --batches 256,1024,4096,16384 --calls 40 > $out/base_$i.json 2>> $out/err.log
  HPSB_LIB_VARIANT=prev timeout 900 python tools/bench_cfg3.py --keys-per-table 400000 --batches 256,1024,4096,16384 --calls 40 > $out/prev_$i.json 2>> $out/err.log
done
for f in $out/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', [(p['batch'], round(p['table_lookup_p50_us'],1), round(p['sample_batch_26_tables_group_one_launch_p50_us'],1), round(p['mean_unique_hit_rate'],3)) for p in d['per_batch']])"; done > $out/summary.txt
cat $out/summary.txt
