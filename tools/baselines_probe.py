"""Timing + agreement probe for the comparison objectives:
one PointwiseL1 epoch and one ListMLE epoch on gen(8192, seed 21) (the C2
dataset), GPU engine vs the reference library on this host.

    python tools/baselines_probe.py
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle.bind import Extractor as OEx, Ref  # noqa: E402
from paper_2510_03243_b200 import Context, Extractor  # noqa: E402


def main():
    import torch
    ref = Ref()
    ctx = Context(0)
    ds = ref.synthesize(8192, 21)
    ids = ds.ids()
    ex = Extractor.make()
    f = ctx.extract(ex, ds.text, ds.offs)
    out = {}
    target = np.log1p(ds.output_len.astype(np.float64))
    order = np.random.default_rng(0).permutation(8192).astype(np.uint32)
    lists = np.stack([np.random.default_rng(i).choice(8192, 10, replace=False)
                      for i in range(2000)]).astype(np.uint32).ravel()
    for name, fn in (("pointwise_epoch", lambda: ctx.pointwise_epoch(f, order, target, 128, 0.1,
                                                                    np.zeros(4096))),
                     ("listmle_epoch", lambda: ctx.listmle_epoch(f, lists, 10, 128, 0.1,
                                                                 np.zeros(4096)))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        out[name + "_ms"] = 1e3 * min(ts)
    for obj, name in ((1, "pointwise_l1"), (2, "listwise_listmle")):
        t0 = time.perf_counter()
        rw, rb, rlt = ref.train(ds, OEx.make(), objective=obj, epochs=1, seed=21)
        out[name + "_ref_train_ms"] = 1e3 * (time.perf_counter() - t0)
        t0 = time.perf_counter()
        w, b, lt = ctx.train_baseline(ex, ds.text, ds.offs, ds.output_len, ids, name, epochs=1,
                                      seed=21)
        out[name + "_gpu_train_ms"] = 1e3 * (time.perf_counter() - t0)
        out[name + "_bit_identical"] = bool((w.view(np.uint64) == rw.view(np.uint64)).all()
                                            and lt[0] == rlt[0] and b == rb)
        out[name + "_max_w_rel"] = float(np.abs(w - rw).max() / np.abs(rw).max())
        out[name + "_loss_rel"] = float(abs(lt[0] - rlt[0]) / abs(rlt[0]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
