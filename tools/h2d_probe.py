"""Pinned host->device copy bandwidth on this box (the e2e ceiling): one
stream, two streams, chunk sizes."""
import time

import torch

n = 2_000_000_000
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for chunk in (16 << 20, 64 << 20, 256 << 20):
    for streams in (1, 2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k, off in enumerate(range(0, n, chunk)):
            st = s1 if streams == 1 or k % 2 == 0 else s2
            with torch.cuda.stream(st):
                d[off:off + chunk].copy_(h[off:off + chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"chunk {chunk >> 20} MB, {streams} stream(s): {n / dt / 1e9:.1f} GB/s")
