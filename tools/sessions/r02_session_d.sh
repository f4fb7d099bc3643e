#!/bin/bash
# replace v3 (64-bit set entries, L2 prefetch from the bin kernel, persistent pipelined set kernel)
tag=${1:-r02d}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_cache_gpu.py -x -q -m gpu > $out/pytest_cache.log 2>&1; echo "rc=$?" >> $out/pytest_cache.log
timeout 300 python tools/bench_replace.py --check > $out/replace.json 2> $out/replace.err; echo "rc=$?" >> $out/replace.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/replace_launches.csv python tools/bench_replace.py --reps 3 > $out/ncu_replace.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_replace_sets -s 20 -c 1 -o $out/replace_sets python tools/bench_replace.py --reps 3 > $out/ncu_full.log 2>&1
timeout 600 python tools/bench_pdb.py --keys 2000000 > $out/pdb.json 2> $out/pdb.err
ls -la $out
