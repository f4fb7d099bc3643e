#!/bin/bash
# source-level ncu of the exact replace's set kernel and bin kernel (engine-fill shape)
tag=${1:-r02cc}
out=gpurun_out/$tag; mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_replace_sets|k_replace_bin" -s 80 -c 2 -o $out/repl python tools/bench_replace.py --reps 20 > $out/ncu.log 2>&1
tail -5 $out/ncu.log
