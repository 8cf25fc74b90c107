"""Where one C2 epoch's time goes (extract / free / build_pairs / SGD)."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import paper_2510_03243_b200 as P  # noqa: E402

ctx = P.Context(0)
ex = P.Extractor.make()
d2 = P.Workload.synthesize(8192, 21)
te, tf = [], []
for _ in range(6):
    t0 = time.perf_counter()
    f = ctx.extract(ex, d2.text, d2.offsets)
    t1 = time.perf_counter()
    f.free()
    t2 = time.perf_counter()
    te.append(t1 - t0)
    tf.append(t2 - t1)
f = ctx.extract(ex, d2.text, d2.offsets)
tb, ts, tt = [], [], []
for _ in range(5):
    t0 = time.perf_counter()
    a, b, y, _ = P.build_pairs(d2.output_len, 0.2, 100000, 12345)
    t1 = time.perf_counter()
    ctx.sgd_epoch(f, a, b, y, 128, 0.1, 1.0, np.zeros(4096))
    t2 = time.perf_counter()
    ctx.train_pairwise(ex, d2.text, d2.offsets, d2.output_len, seed=21, epochs=1)
    t3 = time.perf_counter()
    tb.append(t1 - t0)
    ts.append(t2 - t1)
    tt.append(t3 - t2)
m = lambda v: 1e3 * float(np.median(v[1:]))  # noqa: E731
print(f"extract {m(te):.2f} ms, free {m(tf):.2f} ms, build_pairs(host) {m(tb):.2f} ms, "
      f"sgd_epoch {m(ts):.2f} ms, train_pairwise(1 epoch) {m(tt):.2f} ms")
