#!/bin/bash
# host-side scatter of the sync branch: engine + drop-in tests, bench line (e2e legs)
tag=${1:-r02o}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_dropin.py tests/test_relaxed_gpu.py tests/test_sharded.py -x -q -m gpu > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench20.json 2> $out/bench20.err; echo "rc=$?" >> $out/bench20.err
HPSB_ENGINE_TRACE=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-sweep --no-online --no-cpu-baseline --hit 0.5 > $out/bench_h05.json 2> $out/bench_h05.err
ls -la $out
