#!/bin/bash
# replace A/B: set kernel with the next set's state staged by cp.async (pipe),
# + direct-indexed set table in the bin kernel (pipedir), vs base
tag=${1:-r02ax}
out=gpurun_out/$tag; mkdir -p $out
HPSB_LIB_VARIANT=pipedir timeout 900 python -m pytest tests/test_cache_gpu.py tests/test_engine_gpu.py tests/test_headline_gpu.py -x -q -m gpu > $out/pytest_pipedir.log 2>&1; echo "rc=$?" >> $out/pytest_pipedir.log
for i in 1 2; do
  for v in base pipe pipedir; do
    if [ $v = base ]; then timeout 300 python tools/bench_replace.py --check > $out/${v}_$i.json 2>> $out/err.log;
    else HPSB_LIB_VARIANT=$v timeout 300 python tools/bench_replace.py --check > $out/${v}_$i.json 2>> $out/err.log; fi
  done
done
for f in $out/*_[12].json; do echo "$f: $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print({k: v for k, v in d.items() if 'us' in k or 'check' in k})")"; done > $out/summary.txt
HPSB_LIB_VARIANT=pipedir timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/pipedir_launches.csv python tools/bench_replace.py --reps 3 > $out/ncu.log 2>&1
cat $out/summary.txt
