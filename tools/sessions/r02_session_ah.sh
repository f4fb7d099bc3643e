#!/bin/bash
# e2e host-side A/B: output chunk size and copy threads (pageable + drop-in legs)
tag=${1:-r02ah}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_dropin.py -x -q -m gpu > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
run() { env $2 timeout 600 python bench.py --steps 20 --warmup 5 --no-sweep --no-online --no-cpu-baseline > $out/b_$1.json 2>> $out/err.log; }
for i in 1 2; do
  run base_$i ""
  run s21_$i "HPSB_OUT_CHUNK_SHIFT=21"
  run t12_$i "HPSB_COPY_THREADS=12"
  run t16_$i "HPSB_COPY_THREADS=16"
done
for f in $out/b_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); e=d['e2e']
print('$f', round(e['value']/1e6,1), round(e['pageable']['value']/1e6,1), round(e['pageable']['p50_call_us']), round(e['sync_h050']['value']/1e6,1), round(e['dropin_cpp']['value']/1e6,1))"; done > $out/summary.txt
cat $out/summary.txt
