#!/bin/bash
# cfg 5 (1B-key table, 200M-slot replica) with the read-first miss claims: 300 and 2,000 steps
tag=${1:-r02ch}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python tools/bench_cfg5.py --steps 300 > $out/cfg5_300.json 2> $out/cfg5_300.err
timeout 900 python tools/bench_cfg5.py --steps 2000 > $out/cfg5_2000.json 2> $out/cfg5_2000.err
tail -c 600 $out/cfg5_300.json; tail -c 600 $out/cfg5_2000.json
