#!/bin/bash
# validation: all GPU tests, smoke, bench 20 / 2000 steps
tag=${1:-r02af}
out=gpurun_out/$tag; mkdir -p $out
timeout 1500 python -m pytest tests -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "rc=$?" >> $out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench20.json 2> $out/bench20.err; echo "rc=$?" >> $out/bench20.err
timeout 600 python bench.py --steps 2000 --warmup 20 --no-e2e --no-cpu-baseline --no-online > $out/bench2000.json 2> $out/bench2000.err
ls -la $out
