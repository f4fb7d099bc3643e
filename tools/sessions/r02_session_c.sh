#!/bin/bash
# replace rewrite (touched-set list) + drop-in e2e + sync leg timings
tag=${1:-r02c}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_cache_gpu.py tests/test_headline_gpu.py -x -q -m gpu > $out/pytest_cache.log 2>&1; echo "rc=$?" >> $out/pytest_cache.log
timeout 300 python tools/bench_replace.py --check > $out/replace.json 2> $out/replace.err; echo "rc=$?" >> $out/replace.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/replace_launches.csv python tools/bench_replace.py --reps 3 > $out/ncu_replace.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench20.json 2> $out/bench20.err; echo "rc=$?" >> $out/bench20.err
timeout 1500 python -m pytest tests -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
ls -la $out
