#!/usr/bin/env python
"""Host <-> device copy rates of this box (the ceiling of bench.py's e2e line): pinned
256 MiB buffers, H2D alone, D2H alone and both directions at once (two streams), CUDA events,
mean of 10 after 3 warm-ups.  One JSON line per case."""
from __future__ import annotations

import json


def main():
    import torch

    dev = torch.device("cuda:0")
    n = 256 << 20
    h_a = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_b = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(n, dtype=torch.uint8, device=dev)
    d_b = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def run(h2d: bool, d2h: bool, reps: int):
        for _ in range(reps):
            if h2d:
                with torch.cuda.stream(s1):
                    d_a.copy_(h_a, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    h_b.copy_(d_b, non_blocking=True)

    for name, h2d, d2h in (("h2d", True, False), ("d2h", False, True), ("both", True, True)):
        run(h2d, d2h, 3)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream(dev)
        e0.record(cur)
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        run(h2d, d2h, 10)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
        e1.record(cur)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / 10
        print(json.dumps({"case": name, "bytes_each_direction": n, "ms": round(ms, 4),
                          "gb_s_each_direction": round(n / (ms / 1e3) / 1e9, 2)}))


if __name__ == "__main__":
    main()
