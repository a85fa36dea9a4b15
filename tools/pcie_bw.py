#!/usr/bin/env python
"""Host<->device copy bandwidth of this box (pinned memory): H2D, D2H, both at once."""
import time

import torch

N = 512 << 20
h_a = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h_b = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(N, dtype=torch.uint8, device="cuda")
d_b = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, parts=1, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if h2d:
            with torch.cuda.stream(s1):
                d_a.copy_(h_a, non_blocking=True)
        if d2h:
            step = N // parts
            for k in range(parts):
                with torch.cuda.stream(s2 if k % 2 == 0 else torch.cuda.current_stream()):
                    h_b[k * step:(k + 1) * step].copy_(d_b[k * step:(k + 1) * step], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


for name, a, b, p in [("h2d", 1, 0, 1), ("d2h", 0, 1, 1), ("d2h 2 streams", 0, 1, 2), ("both", 1, 1, 1)]:
    t = run(a, b, p)
    print(f"{name:16s} {t * 1e3:7.2f} ms  {N * (a + b) / t / 1e9:6.1f} GB/s total")
