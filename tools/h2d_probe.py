#!/usr/bin/env python3
"""Pinned host -> device copy bandwidth (the e2e ceiling): one stream and two concurrent
streams.  Profiling tool."""
import time

import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.float16, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.float16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    one = 2 * n / (time.perf_counter() - t) / 1e9
    t = time.perf_counter()
    with torch.cuda.stream(s1):
        d[: n // 2].copy_(h[: n // 2], non_blocking=True)
    with torch.cuda.stream(s2):
        d[n // 2:].copy_(h[n // 2:], non_blocking=True)
    torch.cuda.synchronize()
    two = 2 * n / (time.perf_counter() - t) / 1e9
    print(f"H2D 2 GiB: one stream {one:.1f} GB/s, two streams {two:.1f} GB/s", flush=True)
