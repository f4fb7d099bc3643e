#!/bin/bash
# replace: bin block aggregation + set-state L2 prefetch (A/B vs variants), parity of replace paths; bench line
tag=${1:-r02j}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_cache_gpu.py tests/test_relaxed_gpu.py -x -q -m gpu > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for v in base nopf old base; do
  if [ $v = base ]; then timeout 600 python tools/bench_replace.py --reps 40 >> $out/replace_$v.json 2>> $out/replace.err;
  else HPSB_LIB_VARIANT=$v timeout 600 python tools/bench_replace.py --reps 40 > $out/replace_$v.json 2>> $out/replace.err; fi
done
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench20.json 2> $out/bench20.err; echo "rc=$?" >> $out/bench20.err
ls -la $out
