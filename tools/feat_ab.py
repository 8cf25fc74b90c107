"""A/B timing (argv: n_prompts [filler|random6]) + exactness of the featurize kernels on C4-shaped prompts.

Runs in one process per kernel (PARS_FEAT_V1=1 selects the round-1 kernel):
  python tools/feat_ab.py [n_prompts]
prints one JSON line: kernel ms per launch (CUDA events, device-resident
inputs, 1M-prompt equivalent), exact-score parity against the oracle on a
sample, and fast-mode agreement."""
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2510_03243_b200 as P  # noqa: E402
from oracle.bind import Extractor as OEx  # noqa: E402
from oracle.bind import Oracle  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
pad_words = sys.argv[2] if len(sys.argv) > 2 else "filler"  # "random6": the C4 hard variant
wl = P.Workload.synthesize(n, 31, pad_tokens=512, pad_seed=5, pad_words=pad_words)
w = np.random.default_rng(1234).normal(size=4096) * 0.05
ctx = P.Context(0)
ex = P.Extractor.make()
dev = torch.device("cuda", 0)
d_text = torch.from_numpy(wl.text[: wl.offsets[-1]]).to(dev)
d_offs = torch.from_numpy(wl.offsets).to(dev)
d_w = torch.from_numpy(w).to(dev)
d_s = torch.empty(n, dtype=torch.float64, device=dev)
L = P.lib()
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
out = {"pad_words": pad_words, "bytes_per_prompt": float(wl.offsets[-1]) / n, "kernel": "v1" if os.environ.get("PARS_FEAT_V1") == "1" else ("lane-unfused" if os.environ.get("PARS_FEAT_UNFUSED") == "1" else "lane-fused"), "prompts": n}
for mode, name in ((P.MODE_EXACT, "exact"), (P.MODE_FAST, "fast")):
    def run():
        rc = L.pars_dev_score_text(ctx.h, C.byref(ex), d_text.data_ptr(), d_offs.data_ptr(), n,
                                   d_w.data_ptr(), 0.0, mode, d_s.data_ptr(), st.cuda_stream)
        assert rc == 0, L.pars_last_error()
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = 10
    a.record(st)
    for _ in range(k):
        run()
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / k
    s = d_s.cpu().numpy()
    out[name + "_ms"] = ms
    out[name + "_ms_per_1M"] = ms * 1e6 / n
    if mode == P.MODE_EXACT:
        m = min(n, 20000)
        so = Oracle().score_batch(OEx.make(), wl.text, wl.offsets[: m + 1], w, 0.0, threads=os.cpu_count())
        out["exact_bitexact_sample"] = bool((s[:m].view(np.uint64) == so.view(np.uint64)).all())
        out["exact_sample"] = m
        exact = s.copy()
    else:
        out["fast_max_abs_diff"] = float(np.abs(s - exact).max())
print(json.dumps(out))
