#!/bin/bash
# cost attribution after the read-first miss claims (HPSB_DIAG_SKIP: 1 no stamps, 2 no miss claims, 4 no copy)
tag=${1:-r02cj}
out=gpurun_out/$tag; mkdir -p $out
for h in 0.5 0.9; do
  for sk in 0 1 2 4 3; do
    HPSB_DIAG_SKIP=$sk timeout 300 python bench.py --steps 200 --warmup 5 --hit $h --no-sweep --no-e2e --no-cpu-baseline --no-online > $out/h${h}_s$sk.json 2>> $out/err.log
    python -c "import json; d=json.loads(open('$out/h${h}_s$sk.json').read().strip().splitlines()[-1]); print('h $h skip $sk', round(d['ms_per_step']*1e3,2), 'us/step', round(d['value']/1e9,2))" >> $out/summary.txt
  done
done
cat $out/summary.txt
