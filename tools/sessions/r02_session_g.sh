#!/bin/bash
# relaxed replace mode: its GPU tests, the replace bench (exact vs relaxed), bench line (drop-in leg)
tag=${1:-r02g}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_relaxed_gpu.py -x -q -m gpu > $out/pytest_relaxed.log 2>&1; echo "rc=$?" >> $out/pytest_relaxed.log
timeout 600 python tools/bench_replace.py > $out/replace.json 2> $out/replace.err
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench20.json 2> $out/bench20.err; echo "rc=$?" >> $out/bench20.err
ls -la $out
