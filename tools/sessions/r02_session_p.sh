#!/bin/bash
# exact replace with lane groups (2 sets per warp): parity + A/B vs prev
tag=${1:-r02p}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_cache_gpu.py tests/test_headline_gpu.py tests/test_engine_gpu.py -x -q -m gpu > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for v in base prev base prev; do
  if [ $v = base ]; then timeout 600 python tools/bench_replace.py --reps 40 >> $out/replace_$v.json 2>> $out/replace.err;
  else HPSB_LIB_VARIANT=$v timeout 600 python tools/bench_replace.py --reps 40 >> $out/replace_$v.json 2>> $out/replace.err; fi
done
timeout 600 python tools/bench_replace.py --reps 40 --check > $out/replace_check.json 2>> $out/replace.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_replace_sets<" -s 34 -c 1 \
  -o $out/sets python tools/bench_replace.py --reps 2 > $out/ncu_sets.log 2>&1
ls -la $out
