#!/bin/bash
# Round-2 GPU session: new GPU tests first, full GPU suite, smoke, replace bench, bench (20 and 2000 steps), replace launch list.
tag=${1:-r02a}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi > $out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests/test_headline_gpu.py tests/test_engine_gpu.py tests/test_cache_gpu.py -x -q -m gpu > $out/pytest_new.log 2>&1; echo "rc=$?" >> $out/pytest_new.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "rc=$?" >> $out/smoke.log
timeout 300 python tools/bench_replace.py --check > $out/replace.json 2> $out/replace.err; echo "rc=$?" >> $out/replace.err
timeout 600 python bench.py --steps 20 --warmup 5 > $out/bench20.json 2> $out/bench20.err; echo "rc=$?" >> $out/bench20.err
timeout 600 python bench.py --steps 2000 --warmup 20 --no-e2e --no-cpu-baseline --no-online > $out/bench2000.json 2> $out/bench2000.err; echo "rc=$?" >> $out/bench2000.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/replace_launches.csv python tools/bench_replace.py --reps 3 > $out/ncu_replace.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
ls -la $out
