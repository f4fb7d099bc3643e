#!/bin/bash
# replace A/B: row-prefetch ring in the set kernel (new default) vs the same loop
# without the ring (ring0) vs the committed library (base)
tag=${1:-r02cb}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_cache_gpu.py tests/test_engine_gpu.py tests/test_relaxed_gpu.py -x -q -m gpu > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for i in 1 2 3; do
  for v in new base ring0; do
    if [ $v = new ]; then timeout 300 python tools/bench_replace.py --check > $out/${v}_$i.json 2>> $out/err.log;
    else HPSB_LIB_VARIANT=$v timeout 300 python tools/bench_replace.py --check > $out/${v}_$i.json 2>> $out/err.log; fi
  done
done
for f in $out/*_[123].json; do echo "$f: $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print({k: v for k, v in d.items() if 'fill_us' in k or 'equal' in k or 'user_us' in k})")"; done > $out/summary.txt
cat $out/summary.txt; tail -3 $out/pytest.log
