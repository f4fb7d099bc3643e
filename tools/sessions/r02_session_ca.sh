#!/bin/bash
# fill / drain of the 20-step timed graph: per-call timeline (HPSB_TRACE) of
# 20-step graphs vs the 200-step steady state; the lone-call timeline
tag=${1:-r02ca}
out=gpurun_out/$tag; mkdir -p $out
for i in 1 2; do
  timeout 300 python tools/trace_lookup.py --steps 20 --per-call > $out/trace20_$i.txt 2>&1
done
timeout 300 python tools/trace_lookup.py --steps 200 > $out/trace200.txt 2>&1
timeout 300 python tools/trace_lookup.py --steps 50 --isolated > $out/isolated.txt 2>&1
timeout 300 python tools/bench_replace.py --check > $out/replace.json 2> $out/replace.err
cat $out/trace20_1.txt $out/trace200.txt $out/isolated.txt
