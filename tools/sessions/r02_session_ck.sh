#!/bin/bash
# lookup A/B: miss-table key array read with the entry (KEYTAB, default) vs read-first without it (kt0)
tag=${1:-r02ck}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_headline_gpu.py tests/test_engine_gpu.py tests/test_cache_gpu.py tests/test_relaxed_gpu.py tests/test_sharded.py -x -q -m gpu > $out/pytest_kt0.log 2>&1; echo "rc=$?" >> $out/pytest_kt0.log
for i in 1 2 3; do
  for v in def kt0; do
    for s in 200 20; do
      if [ $v = def ]; then timeout 300 python bench.py --steps $s --warmup 10 --no-e2e --no-online --no-cpu-baseline > $out/${v}_${s}_$i.json 2>> $out/err.log;
      else HPSB_LIB_VARIANT=$v timeout 300 python bench.py --steps $s --warmup 10 --no-e2e --no-online --no-cpu-baseline > $out/${v}_${s}_$i.json 2>> $out/err.log; fi
    done
  done
done
for f in $out/*_[123].json; do echo "$f: $(python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); sw=d.get('hit_rate_sweep',{})
print({k: round(v['keys_per_s']/1e9,3) for k,v in sw.items()}, 'ok' if d.get('self_check',{}).get('ok', True) else 'CHECK-FAIL')")"; done > $out/summary.txt
cat $out/summary.txt; tail -2 $out/pytest_kt0.log
