#!/bin/bash
# ncu evidence for the round (under gpurun, 1 GPU): launch list of the bench
# workload, a full capture of the lookup kernel, and full captures of the
# update / dump kernels at the Table-3 1 GB size.
tag=${1:-prof}
out=gpurun_out/$tag; mkdir -p $out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 20 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline --no-online > $out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lookup_tag -s 40 -c 2 \
  -o $out/prof python bench.py --steps 20 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline --no-online > $out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_update_probe|k_update_write|k_dump_keys" -s 2 -c 3 \
  -o $out/prof_cacheapi python tools/bench_table3.py --sizes 1 --reps 2 > $out/ncu_cacheapi.log 2>&1
ls -la $out
