"""C2-shaped SGD epoch timing + exactness (8,192 prompts, 100k pairs, batch
128, 782 steps): median wall time of ctx.sgd_epoch(algo="cluster") over 7
calls (the epoch kernel dominates; inputs stay resident in the Features
handle), and the weights / loss / active count bit-compared with the oracle.
  python tools/sgd_ab.py          (PARS_CUDA_LIB selects a variant build)"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2510_03243_b200 as P  # noqa: E402
from oracle.bind import Oracle  # noqa: E402

ctx = P.Context(0)
ex = P.Extractor.make()
wl = P.Workload.synthesize(8192, 21)
f = ctx.extract(ex, wl.text, wl.offsets)
a, b, y, _ = P.build_pairs(wl.output_len, 0.2, 100000, 12345)
w0 = np.random.default_rng(5).normal(size=4096) * 0.01
ts = []
for _ in range(7):
    t0 = time.perf_counter()
    w, el, act = ctx.sgd_epoch(f, a, b, y, 128, 0.1, 1.0, w0, algo="cluster")
    ts.append(time.perf_counter() - t0)
rp, idx, val = f.download()
ow, oel, oact = Oracle().sgd_epoch(rp, idx, val, 4096, a, b, y, 128, 0.1, 1.0, w0)
print(json.dumps({"epoch_ms": 1e3 * float(np.median(ts)), "min_ms": 1e3 * min(ts),
                  "bit_identical": bool(act == oact and el.hex() == oel.hex()
                                        and (w.view(np.uint64) == ow.view(np.uint64)).all()),
                  "steps": -(-len(a) // 128)}))
