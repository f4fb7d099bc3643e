#!/bin/bash
# A/B the lookup kernel variants (measurement only). Usage under gpurun:
#   bash tools/ab.sh <tag> "ENV=.. ENV2=.." "ENV=.." ...
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
i=0
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-sweep --no-online --steps 1000 > $out/ab_$i.json 2>> $out/ab.err
  python - "$cfg" $out/ab_$i.json <<'PY' >> $out/ab.txt
import json, sys
d = json.loads(open(sys.argv[2]).read().splitlines()[0])
print(f"{sys.argv[1]:40s} keys/s {d['value']/1e9:6.3f} G  step {d['ms_per_step']*1e3:6.2f} us  kernel {d['roofline']['kernel_us']:6.2f} us  p50 {d['p50_batch_latency_us']:6.2f} us  h {d['measured_unique_hit_rate']:.3f}")
PY
  i=$((i+1))
done
cat $out/ab.txt
