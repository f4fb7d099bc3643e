#!/bin/bash
# engine side stream + pageable output + drop-in VDB: GPU tests, acceptance, bench with the e2e legs
tag=${1:-r02b}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_dropin.py -x -q -m gpu > $out/pytest_engine.log 2>&1; echo "rc=$?" >> $out/pytest_engine.log
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench20.json 2> $out/bench20.err; echo "rc=$?" >> $out/bench20.err
timeout 1500 python -m pytest tests -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
ls -la $out
