#!/bin/bash
tag=${1:-r02aa}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_cache_gpu.py tests/test_engine_gpu.py -x -q -m gpu > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 900 python tools/bench_table3.py > $out/table3.json 2> $out/table3.err
ls -la $out
