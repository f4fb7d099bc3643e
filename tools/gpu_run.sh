#!/bin/bash
# One GPU session: parity tests, bench, launch list and a full ncu capture of the lookup kernel.
# Usage (under gpurun): bash tools/gpu_run.sh [tag] [skip-tests]
tag=${1:-run}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi > $out/nvsmi.txt 2>&1
if [ "$2" != "skip-tests" ]; then
  timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
fi
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" >> $out/bench.err
for v in ${AB_VARIANTS:-}; do
  HPSB_LOOKUP_KERNEL=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-sweep > $out/bench_$v.json 2>> $out/bench.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 20 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline --no-online > $out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lookup_tag -s 40 -c 2 \
  -o $out/prof python bench.py --steps 20 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline --no-online > $out/ncu_full.log 2>&1
ls -la $out
