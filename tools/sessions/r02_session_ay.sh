#!/bin/bash
# replace A/B: direct-indexed set table in bin (dir), per-key slab meta from bin + 32-bit eviction argmin (fast), both (dirfast) vs base
tag=${1:-r02ax}
out=gpurun_out/$tag; mkdir -p $out
HPSB_LIB_VARIANT=dirfast timeout 900 python -m pytest tests/test_cache_gpu.py tests/test_engine_gpu.py tests/test_headline_gpu.py -x -q -m gpu > $out/pytest_dirfast.log 2>&1; echo "rc=$?" >> $out/pytest_dirfast.log
for i in 1 2; do
  for v in base dir fast dirfast; do
    if [ $v = base ]; then timeout 300 python tools/bench_replace.py --check > $out/${v}_$i.json 2>> $out/err.log;
    else HPSB_LIB_VARIANT=$v timeout 300 python tools/bench_replace.py --check > $out/${v}_$i.json 2>> $out/err.log; fi
  done
done
for f in $out/*_[12].json; do echo "$f: $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print({k: v for k, v in d.items() if 'us' in k or 'check' in k})")"; done > $out/summary.txt
HPSB_LIB_VARIANT=dirfast timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/dirfast_launches.csv python tools/bench_replace.py --reps 3 > $out/ncu.log 2>&1
cat $out/summary.txt
