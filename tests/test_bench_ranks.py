"""The multi-rank (replica) measurement path of bench.py on CPU: two gloo
ranks, the job time is the max over ranks (the slowest replica defines the
whole-job throughput)."""
import os
import socket
import sys
from pathlib import Path

import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    import bench

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = 10.0 + 7.5 * rank
        q.put((rank, bench.max_over_ranks(mine, dist, "cpu")))
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    got = dict(q.get() for _ in range(2))
    assert all(p.exitcode == 0 for p in ps)
    assert got == {0: 17.5, 1: 17.5}


def test_max_over_ranks_single_process_is_identity():
    sys.path.insert(0, str(ROOT))
    import bench

    assert bench.max_over_ranks(3.25, None, "cpu") == 3.25


def test_cpu_replica_baseline_runs_n_concurrent_reference_engines():
    """N > 1: the CPU baseline is N independent reference replicas served
    concurrently, value = their aggregate keys/s."""
    import types

    import pytest

    sys.path.insert(0, str(ROOT))
    import bench
    import oracle

    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    wl = bench.Workload(keyspace=100_000, dim=16, cache_frac=0.2, batch=2048)
    args = types.SimpleNamespace(hit=0.9)
    one = bench.cpu_baseline(args, wl, replicas=1)
    two = bench.cpu_baseline(args, wl, replicas=2)
    assert one["value"] > 0 and two["value"] > 0, (one, two)
    assert two["replicas"] == 2 and one["replicas"] == 1
    assert two["kind"] == "reference" and "2 concurrent reference" in two["sample"]
