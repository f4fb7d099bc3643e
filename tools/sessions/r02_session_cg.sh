#!/bin/bash
# validation: peer lookup with read-first stamps + warp-aggregated inbox appends
# (sharded GPU tests, memcheck of the peer smoke, the 2-rank peer bench), full GPU
# suite, and the driver-shaped bench line (20 steps) with the capped sync leg
tag=${1:-r02cg}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
timeout 600 compute-sanitizer --tool memcheck python tools/peer_smoke.py > $out/memcheck_peer.log 2>&1; echo "rc=$?" >> $out/memcheck_peer.log
timeout 300 python tools/bench_peer.py --world 2 > $out/peer2.json 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > $out/bench20.json 2> $out/bench20.err; echo "rc=$?" >> $out/bench20.err
tail -2 $out/pytest_gpu.log; tail -3 $out/memcheck_peer.log; tail -2 $out/peer2.json
