#!/bin/bash
# block-published claims: lookup parity + A/B at h 0.5 / 0.9 (200 and 20 steps)
tag=${1:-r02am}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_cache_gpu.py tests/test_headline_gpu.py tests/test_engine_gpu.py -x -q -m gpu > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for i in 1 2; do
  for v in base prev; do
    for h in 0.5 0.9; do
      for st in 200 20; do
        if [ $v = base ]; then timeout 300 python bench.py --steps $st --warmup 5 --hit $h --no-sweep --no-e2e --no-cpu-baseline --no-online > $out/${v}_h${h}_s${st}_$i.json 2>> $out/err.log;
        else HPSB_LIB_VARIANT=prev timeout 300 python bench.py --steps $st --warmup 5 --hit $h --no-sweep --no-e2e --no-cpu-baseline --no-online > $out/${v}_h${h}_s${st}_$i.json 2>> $out/err.log; fi
        python -c "import json; d=json.loads(open('$out/${v}_h${h}_s${st}_$i.json').read().strip().splitlines()[-1]); print('$v h $h steps $st rep $i', round(d['ms_per_step']*1e3,2), 'us/step', round(d['value']/1e9,3), 'check', d['self_check']['ok'])" >> $out/summary.txt
      done
    done
  done
done
cat $out/summary.txt
