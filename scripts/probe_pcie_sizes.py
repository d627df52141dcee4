#!/usr/bin/env python
"""PCIe copy rates by transfer size (diagnostic for the host-buffer pipeline): a stream of
back-to-back pinned H2D copies of `size` bytes on one stream and D2H copies on another, ~1.5 GB
per direction, alone and at once; prints GB/s per direction (CUDA events, best of 3)."""
import json
import sys

import torch


def main():
    total = 1536 << 20
    h_in = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(total, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(total, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for size in (4 << 20, 8 << 20, 23 << 20, 64 << 20, 256 << 20, total):
        n = total // size

        def up():
            for k in range(n):
                d_a[k * size:(k + 1) * size].copy_(h_in[k * size:(k + 1) * size], non_blocking=True)

        def down():
            for k in range(n):
                h_out[k * size:(k + 1) * size].copy_(d_b[k * size:(k + 1) * size], non_blocking=True)

        def timed(ops):
            best = []
            for _ in range(3):
                torch.cuda.synchronize()
                ev = []
                for st, fn in ops:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    with torch.cuda.stream(st):
                        fn()
                    e1.record(st)
                    ev.append((e0, e1))
                torch.cuda.synchronize()
                best.append(max(a.elapsed_time(b) for a, b in ev))
            return min(best)

        gb = n * size / 1e9
        r = {"size_mb": size >> 20, "copies": n, "h2d_gbs": round(gb / timed([(s1, up)]) * 1e3, 1),
             "d2h_gbs": round(gb / timed([(s2, down)]) * 1e3, 1),
             "bidir_gbs_each": round(gb / timed([(s1, up), (s2, down)]) * 1e3, 1)}
        print(json.dumps(r), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
