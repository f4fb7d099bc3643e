#!/bin/bash
# round-2 re-measurement of the other BASELINE configs: cfg 5 (1B keys, one replica) and cfg 3 (26 tables, full VDB)
tag=${1:-r02r}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python tools/bench_cfg5.py --steps 300 > $out/cfg5.json 2> $out/cfg5.err
timeout 900 python tools/bench_cfg5.py --steps 2000 > $out/cfg5_2000.json 2> $out/cfg5_2000.err
free -g > $out/free.txt
timeout 2400 python tools/bench_cfg3.py > $out/cfg3.json 2> $out/cfg3.err
ls -la $out
