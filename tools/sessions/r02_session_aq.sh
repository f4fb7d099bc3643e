#!/bin/bash
# compute-sanitizer memcheck over the smoke and a cross-section of the GPU tests (small geometries)
tag=${1:-r02aq}
out=gpurun_out/$tag; mkdir -p $out
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_memcheck.log 2>&1; echo "rc=$?" >> $out/smoke_memcheck.log
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -x -q -m gpu \
  tests/test_cache_gpu.py::test_slot_for_slot_state_equals_oracle \
  tests/test_cache_gpu.py::test_replace_small_and_large_batches_slot_exact \
  tests/test_cache_gpu.py::test_lookup_device_geometries_and_edge_keys \
  tests/test_cache_gpu.py::test_online_update_interleaved_with_lookups_stream_ordered \
  tests/test_relaxed_gpu.py tests/test_engine_gpu.py::test_lockstep_with_engine_oracle_power_law \
  tests/test_engine_gpu.py::test_zero_copy_small_calls_pinned_and_pageable_match_oracle \
  tests/test_engine_gpu.py::test_large_pageable_batches_lockstep_with_engine_oracle \
  > $out/tests_memcheck.log 2>&1; echo "rc=$?" >> $out/tests_memcheck.log
ls -la $out
