#!/bin/bash
# drop-in C++ engine: LookupResult storage sized by a background thread (spare
# vector) -- the reference's own unit tests / acceptance over the drop-in, and
# the drop-in e2e leg (3 reps)
tag=${1:-r02ci}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_dropin.py -x -q -m gpu > $out/pytest_dropin.log 2>&1; echo "rc=$?" >> $out/pytest_dropin.log
for i in 1 2 3; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-sweep --no-online --no-cpu-baseline > $out/bench_$i.json 2>> $out/err.log
done
for f in $out/bench_[123].json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); e=d['e2e']
print('$f', round(e['value']/1e6,1), round(e['pageable']['value']/1e6,1), round(e['sync_h050']['value']/1e6,1), {k: v for k, v in e.get('dropin_cpp', {}).items() if not isinstance(v, (list, dict))})"; done > $out/summary.txt
cat $out/summary.txt; tail -2 $out/pytest_dropin.log
