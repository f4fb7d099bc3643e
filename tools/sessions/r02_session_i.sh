#!/bin/bash
# replace kernels: A/B of the relaxed kernel's occupancy, ncu of both replace paths
tag=${1:-r02i}
out=gpurun_out/$tag; mkdir -p $out
timeout 600 python tools/bench_replace.py --reps 20 > $out/replace_base.json 2> $out/replace.err
HPSB_LIB_VARIANT=rm6 timeout 600 python tools/bench_replace.py --reps 20 > $out/replace_rm6.json 2>> $out/replace.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_replace_relaxed|k_replace_sets|k_replace_bin" -c 6 \
  -o $out/repl python tools/bench_replace.py --reps 2 > $out/ncu_repl.log 2>&1
ls -la $out
