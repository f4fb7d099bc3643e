#!/bin/bash
# 20-step headline A/B: the first (unchained) call as the lone-call variant (default) vs the pipelined one
tag=${1:-r02ae}
out=gpurun_out/$tag; mkdir -p $out
for i in 1 2 3; do
  for v in base allp; do
    if [ $v = base ]; then timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-online --no-sweep > $out/b_${v}_$i.json 2>> $out/err.log;
    else HPSB_LOOKUP_ALL_PIPELINED=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-online --no-sweep > $out/b_${v}_$i.json 2>> $out/err.log; fi
  done
done
for f in $out/b_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/1e9,3), round(d['ms_per_step']*1e3,2), d['p50_batch_latency_us'])"; done > $out/summary.txt
cat $out/summary.txt
