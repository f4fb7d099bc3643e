#!/bin/bash
# lookup A/B: miss claims after the row copies (late) vs before (base), h 0.5 / 0.9, 200 and 20 steps
tag=${1:-r02ar}
out=gpurun_out/$tag; mkdir -p $out
HPSB_LIB_VARIANT=late timeout 600 python -m pytest tests/test_headline_gpu.py tests/test_cache_gpu.py -x -q -m gpu > $out/pytest_late.log 2>&1; echo "rc=$?" >> $out/pytest_late.log
for i in 1 2; do
  for v in base late; do
    for h in 0.5 0.9; do
      for st in 200 20; do
        if [ $v = base ]; then timeout 300 python bench.py --steps $st --warmup 5 --hit $h --no-sweep --no-e2e --no-cpu-baseline --no-online > $out/${v}_h${h}_s${st}_$i.json 2>> $out/err.log;
        else HPSB_LIB_VARIANT=late timeout 300 python bench.py --steps $st --warmup 5 --hit $h --no-sweep --no-e2e --no-cpu-baseline --no-online > $out/${v}_h${h}_s${st}_$i.json 2>> $out/err.log; fi
        python -c "import json; d=json.loads(open('$out/${v}_h${h}_s${st}_$i.json').read().strip().splitlines()[-1]); print('$v h $h steps $st rep $i', round(d['ms_per_step']*1e3,2), 'us/step', round(d['value']/1e9,3), 'check', d['self_check']['ok'])" >> $out/summary.txt
      done
    done
  done
done
cat $out/summary.txt
