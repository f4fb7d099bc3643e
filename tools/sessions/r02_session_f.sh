#!/bin/bash
# engine (reserve, native cold tier) tests, full GPU suite, smoke, bench (20 / 2000 steps),
# launch list, full ncu of the timed lookup kernel, whole-graph ncu of the timed stream
tag=${1:-r02f}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi > $out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -m gpu > $out/pytest_engine.log 2>&1; echo "rc=$?" >> $out/pytest_engine.log
timeout 1500 python -m pytest tests -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "rc=$?" >> $out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench20.json 2> $out/bench20.err; echo "rc=$?" >> $out/bench20.err
timeout 600 python bench.py --steps 2000 --warmup 20 --no-e2e --no-cpu-baseline --no-online > $out/bench2000.json 2> $out/bench2000.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 20 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline --no-online > $out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lookup_tag -s 40 -c 1 \
  -o $out/prof python bench.py --steps 20 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline --no-online > $out/ncu_full.log 2>&1
timeout 900 ncu --graph-profiling graph --clock-control none \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed \
  --csv --log-file $out/graph.csv python tools/trace_lookup.py --steps 200 --no-trace > $out/ncu_graph.log 2>&1
ls -la $out
