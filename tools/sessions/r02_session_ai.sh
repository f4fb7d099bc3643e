#!/bin/bash
# host-side scatter for zero-copy sync calls: engine tests, cfg 1 engine vs reference, cfg3 per-table latency
tag=${1:-r02ai}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_dropin.py tests/test_sharded.py -x -q -m gpu > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 900 python tools/bench_cfg1.py > $out/cfg1.json 2> $out/cfg1.err
ls -la $out
