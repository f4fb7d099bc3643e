#!/bin/bash
# new replace default (dirfast): full GPU tests + smoke; replace A/B vs m5 (5 blocks/SM) and old (round-2 state)
tag=${1:-r02az}
out=gpurun_out/$tag; mkdir -p $out
timeout 1200 python -m pytest tests -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "rc=$?" >> $out/smoke.log
for i in 1 2; do
  for v in new m5 old; do
    if [ $v = new ]; then timeout 300 python tools/bench_replace.py --check > $out/${v}_$i.json 2>> $out/err.log;
    else HPSB_LIB_VARIANT=$v timeout 300 python tools/bench_replace.py --check > $out/${v}_$i.json 2>> $out/err.log; fi
  done
done
for f in $out/*_[12].json; do echo "$f: $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print({k: v for k, v in d.items() if 'us' in k or 'equal' in k})")"; done > $out/summary.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/new_launches.csv python tools/bench_replace.py --reps 3 > $out/ncu.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $out/bench20.json 2> $out/bench20.err; echo "rc=$?" >> $out/bench20.err
cat $out/summary.txt
