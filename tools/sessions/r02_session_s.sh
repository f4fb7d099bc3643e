#!/bin/bash
tag=${1:-r02s}
out=gpurun_out/$tag; mkdir -p $out
timeout 600 python -m pytest tests/test_relaxed_gpu.py -x -q -m gpu > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 300 python tools/ubench_d2h.py > $out/d2h.json 2> $out/d2h.err
ls -la $out
