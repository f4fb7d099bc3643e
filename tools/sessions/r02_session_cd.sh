#!/bin/bash
# replace A/B: scan mode (dense direct-indexed calls walk the set table, no
# touched-set list) = new default, vs HPSB_REPL_SCAN=0 (same library, list
# mode) vs the committed library (base)
tag=${1:-r02cd}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_cache_gpu.py tests/test_engine_gpu.py tests/test_relaxed_gpu.py tests/test_headline_gpu.py -x -q -m gpu > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for i in 1 2 3; do
  timeout 300 python tools/bench_replace.py --check > $out/new_$i.json 2>> $out/err.log
  HPSB_REPL_SCAN=0 timeout 300 python tools/bench_replace.py --check > $out/noscan_$i.json 2>> $out/err.log
  HPSB_LIB_VARIANT=base timeout 300 python tools/bench_replace.py --check > $out/base_$i.json 2>> $out/err.log
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python tools/bench_replace.py --reps 20 > $out/ncu_launch.log 2>&1
for f in $out/*_[123].json; do echo "$f: $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print({k: v for k, v in d.items() if 'fill_us' in k or 'equal' in k or 'user_us' in k})")"; done > $out/summary.txt
cat $out/summary.txt; tail -3 $out/pytest.log
