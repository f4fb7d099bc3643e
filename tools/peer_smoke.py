#!/usr/bin/env python
"""One peer-memory lookup in one process (world 1), step by step, for
diagnosis under compute-sanitizer."""
import faulthandler
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
faulthandler.dump_traceback_later(100, exit=True, file=sys.stderr)


def main():
    import torch
    import torch.distributed as dist

    import paper_2210_08804_b200 as hps
    from paper_2210_08804_b200 import sharded

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("gloo", rank=0, world_size=1)
    cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=64, slabs_per_set=2, dimension=8))
    print("cache", flush=True)
    peer = sharded.PeerShardedLookup(cache, inbox_cap=1 << 14)
    print("group", flush=True)
    keys = torch.arange(100, dtype=torch.int64, device="cuda")
    default = torch.full((8,), -1.0, device="cuda")
    torch.cuda.synchronize()
    out, fl = peer.lookup(keys, default)
    print("launched", flush=True)
    torch.cuda.synchronize()
    print("synced", fl.sum().item(), out[:8].tolist(), flush=True)
    print("drain", len(cache.peer_drain(1 << 14)), flush=True)
    peer.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
