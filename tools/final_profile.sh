#!/bin/bash
# Round-end evidence (under gpurun, 1 GPU): GPU tests, smoke, the bench line,
# the reference arm, the bench's launch list, and full ncu captures of the
# pipelined lookup kernel (k_lookup_tag<8, 8, false>, the timed graph's
# variant), the lone-call variant and the small single-block kernel.
tag=${1:-final}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi > $out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -p no:faulthandler > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" >> $out/bench.err
timeout 600 python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 20 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline --no-online > $out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_lookup_tag<\(int\)8, \(int\)8, \(bool\)0>" -s 3 -c 1 \
  -o $out/prof python bench.py --steps 20 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline --no-online > $out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_lookup_small" -s 20 -c 1 \
  -o $out/prof_small python tools/bench_cfg1.py --batches 200 --thresholds 0.8 > $out/ncu_small.log 2>&1
ls -la $out
