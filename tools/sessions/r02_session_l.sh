#!/bin/bash
# relaxed replace: lane-group variants A/B + tests + ncu; warm refresh in the bench line
tag=${1:-r02l}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_relaxed_gpu.py tests/test_engine_gpu.py -x -q -m gpu > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for v in base g32 mb4 g8 base; do
  if [ $v = base ]; then timeout 600 python tools/bench_replace.py --only relaxed --reps 40 >> $out/relaxed_$v.json 2>> $out/replace.err;
  else HPSB_LIB_VARIANT=$v timeout 600 python tools/bench_replace.py --only relaxed --reps 40 > $out/relaxed_$v.json 2>> $out/replace.err; fi
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_replace_relaxed" -c 2 \
  -o $out/relaxed python tools/bench_replace.py --only relaxed --reps 2 > $out/ncu_relaxed.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench20.json 2> $out/bench20.err; echo "rc=$?" >> $out/bench20.err
ls -la $out
