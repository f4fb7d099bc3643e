#!/bin/bash
tag=${1:-r02v}
out=gpurun_out/$tag; mkdir -p $out
timeout 150 python tools/peer_smoke.py > $out/smoke.log 2>&1; echo "rc=$?" >> $out/smoke.log
timeout 300 compute-sanitizer --tool memcheck python tools/peer_smoke.py > $out/memcheck.log 2>&1; echo "rc=$?" >> $out/memcheck.log
nvidia-smi > $out/nvsmi.txt 2>&1
ls -la $out
