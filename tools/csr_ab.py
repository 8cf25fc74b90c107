"""Timing + exactness of pars_dev_features_score (repeated scoring over
precomputed features) on the 1 M C4 prompts: CUDA events over 10 calls, and
the scores bit-compared with the fused text path's exact scores.
  python tools/csr_ab.py [n]"""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_03243_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
wl = P.Workload.synthesize(n, 31, pad_tokens=512, pad_seed=5)
w = np.random.default_rng(1234).normal(size=4096) * 0.05
ctx = P.Context(0)
ex = P.Extractor.make()
f = ctx.extract(ex, wl.text, wl.offsets)
nnz = int(f.download()[0][-1])
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
d_w = torch.from_numpy(w).to(dev)
out = torch.empty(n, dtype=torch.float64, device=dev)
L = P.lib()


def run():
    assert L.pars_dev_features_score(ctx.h, C.c_void_p(f.h), 0, n, d_w.data_ptr(), 0.0, out.data_ptr(),
                                     st.cuda_stream) == 0, L.pars_last_error()


for _ in range(3):
    run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(10):
    run()
b.record(st)
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
ref = ctx.score_text(ex, wl.text, wl.offsets, w, 0.0)
got = out.cpu().numpy()
moved = nnz * 4 + n * 28
print(json.dumps({"n": n, "nnz": nnz, "ms": ms, "GBps": moved / (ms / 1e3) / 1e9,
                  "bit_identical": bool((got.view(np.uint64) == ref.view(np.uint64)).all())}))
