"""Probe: one C2 training epoch (8,192 prompts, 100k pairs) through the C ABI,
timed per phase (run under ncu for the per-kernel launch list)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_03243_b200 as P  # noqa: E402

ctx = P.Context(0)
ex = P.Extractor.make()
d2 = P.Workload.synthesize(8192, 21)
for k in range(3):
    t0 = time.perf_counter()
    f = ctx.extract(ex, d2.text, d2.offsets)
    t1 = time.perf_counter()
    a, b, y, _ = P.build_pairs(d2.output_len, 0.2, 100000, 12345)
    t2 = time.perf_counter()
    w, el, act = ctx.sgd_epoch(f, a, b, y, 128, 0.1, 1.0, np.zeros(4096))
    t3 = time.perf_counter()
    print(f"extract {1e3*(t1-t0):.2f} ms  build_pairs {1e3*(t2-t1):.2f} ms  sgd_epoch {1e3*(t3-t2):.2f} ms")
    f.free()
