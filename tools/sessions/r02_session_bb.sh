#!/bin/bash
# replace A/B: per-block dynamic item grabs (dyn) vs static strided share (new default)
tag=${1:-r02bb}
out=gpurun_out/$tag; mkdir -p $out
HPSB_LIB_VARIANT=dyn timeout 900 python -m pytest tests/test_cache_gpu.py tests/test_engine_gpu.py -x -q -m gpu > $out/pytest_dyn.log 2>&1; echo "rc=$?" >> $out/pytest_dyn.log
for i in 1 2 3; do
  for v in new dyn; do
    if [ $v = new ]; then timeout 300 python tools/bench_replace.py --check > $out/${v}_$i.json 2>> $out/err.log;
    else HPSB_LIB_VARIANT=$v timeout 300 python tools/bench_replace.py --check > $out/${v}_$i.json 2>> $out/err.log; fi
  done
done
for f in $out/*_[123].json; do echo "$f: $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print({k: v for k, v in d.items() if 'fill_us' in k or 'equal' in k})")"; done > $out/summary.txt
cat $out/summary.txt
