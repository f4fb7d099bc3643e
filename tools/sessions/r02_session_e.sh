#!/bin/bash
# replace A/B variants + sync-branch phase trace
tag=${1:-r02e}
out=gpurun_out/$tag; mkdir -p $out
for v in base a b c d e f; do
  if [ $v = base ]; then e=""; else e="HPSB_LIB_VARIANT=$v"; fi
  env $e timeout 300 python tools/bench_replace.py > $out/replace_$v.json 2>> $out/replace.err
done
HPSB_ENGINE_TRACE=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-sweep --no-online --no-cpu-baseline > $out/bench_trace.json 2> $out/bench_trace.err
ls -la $out
