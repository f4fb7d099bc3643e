#!/bin/bash
# ncu of the relaxed replace kernel + the exact set kernel (warm); host VDB fetch thread sweep
tag=${1:-r02k}
out=gpurun_out/$tag; mkdir -p $out
nproc > $out/nproc.txt; lscpu >> $out/nproc.txt 2>&1; cat /sys/kernel/mm/transparent_hugepage/enabled >> $out/nproc.txt
timeout 600 python tools/vdb_probe.py > $out/vdb.json 2> $out/vdb.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_replace_relaxed<|k_update_probe|k_update_write" -c 4 \
  -o $out/relaxed python tools/bench_replace.py --reps 2 > $out/ncu_relaxed.log 2>&1
ls -la $out
