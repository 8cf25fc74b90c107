"""Small cluster-SGD epoch for compute-sanitizer (racecheck / synccheck /
memcheck): 400 prompts, 1,500 pairs, batch 128 (12 steps, a partial last
step), checked bit-for-bit against the oracle. The full test sizes take
longer than racecheck's budget on the 8-CTA cluster kernel.
  compute-sanitizer --tool racecheck python tools/san_sgd.py"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_03243_b200 as P  # noqa: E402
from oracle.bind import Oracle  # noqa: E402

ctx = P.Context(0)
orc = Oracle()
wl = P.Workload.synthesize(400, 12)
e = P.Extractor.make()
f = ctx.extract(e, wl.text, wl.offsets)
rp, idx, val = f.download()
a, b, y, _ = P.build_pairs(wl.output_len, 0.2, 1500, 99)
w0 = np.random.default_rng(1).normal(size=4096) * 0.01
for algo in ("cluster", "single"):
    w, el, act = ctx.sgd_epoch(f, a, b, y, 128, 0.1, 1.0, w0, algo=algo)
    ow, oel, oact = orc.sgd_epoch(rp, idx, val, 4096, a, b, y, 128, 0.1, 1.0, w0)
    ok = act == oact and el.hex() == oel.hex() and (w.view(np.uint64) == ow.view(np.uint64)).all()
    print(f"sgd {algo}: steps={-(-len(a) // 128)} bit_identical={ok}")
    assert ok
