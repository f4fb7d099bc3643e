#!/bin/bash
# peer-memory sharded lookup: tests (1 and 2 processes on one GPU)
tag=${1:-r02t}
out=gpurun_out/$tag; mkdir -p $out
timeout 600 python -m pytest tests/test_sharded.py -x -q -m gpu -k peer -s > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
ls -la $out
