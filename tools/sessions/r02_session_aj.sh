#!/bin/bash
# group (multi-table) sync path with host scatter: engine tests + cfg 3 small
tag=${1:-r02aj}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_dropin.py -x -q -m gpu > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 1500 python tools/bench_cfg3.py --keys-per-table 400000 --batches 1,16,256,1024,4096 > $out/cfg3_small.json 2> $out/cfg3.err
ls -la $out
