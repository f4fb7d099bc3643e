#!/usr/bin/env python
"""D2H bandwidth of a 33.6 MB result (cfg 2's rows per call) into pinned host
memory: one cudaMemcpyAsync vs the same bytes split over 2 / 4 streams
(copy engines), and H2D for reference. Prints one JSON line."""
import json

import torch


def main():
    n = 65536 * 128 * 4
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    host = torch.empty(n, dtype=torch.uint8).pin_memory()
    streams = [torch.cuda.Stream() for _ in range(4)]
    res = {"bytes": n}

    def run(k, d2h=True, reps=30):
        per = (n + k - 1) // k
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        cur = torch.cuda.current_stream()
        ev0.record(cur)
        for _ in range(reps):
            for i in range(k):
                s = streams[i]
                s.wait_stream(cur)
                with torch.cuda.stream(s):
                    a, b = i * per, min(n, (i + 1) * per)
                    if d2h:
                        host[a:b].copy_(dev[a:b], non_blocking=True)
                    else:
                        dev[a:b].copy_(host[a:b], non_blocking=True)
            for i in range(k):
                cur.wait_stream(streams[i])
        ev1.record(cur)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / reps
        return {"ms": ms, "gbs": n / ms / 1e6}

    for k in (1, 2, 4):
        run(k)
        res[f"d2h_{k}_streams"] = run(k)
    res["h2d_1_stream"] = run(1, d2h=False)
    res["h2d_2_streams"] = run(2, d2h=False)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
