#!/bin/bash
tag=${1:-r02b}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_cache_gpu.py -x -q -m gpu > $out/pytest_cache.log 2>&1; echo "rc=$?" >> $out/pytest_cache.log
timeout 300 python tools/bench_replace.py --check > $out/replace.json 2> $out/replace.err; echo "rc=$?" >> $out/replace.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/replace_launches.csv python tools/bench_replace.py --reps 3 > $out/ncu_replace.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
ls -la $out
