"""Timing + exactness of the priority sort (pars_dev_priority_order) on
1M C4-like keys: device-resident random-normal scores, burst tie ranks
(= index), CUDA events per call; the order is checked against numpy's
stable argsort of the same keys.
  python tools/sort_ab.py [n] [repeat]
repeat r > 1: n / r distinct scores, each repeated ~r times (tie-heavy keys);
repeat 0: distinct scores on only four top 32-bit words (the high-word
speculation's worst case: its fixup falls back to the full LSD)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_03243_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
rng = np.random.default_rng(3)
s = rng.normal(size=n) * 0.3
rep = int(sys.argv[2]) if len(sys.argv) > 2 else 1
if rep > 1:
    s = rng.choice(s[: max(1, n // rep)], size=n)
elif rep == 0:
    s = (1.0 + rng.integers(0, 2**32, size=n) * 2.0**-52) * rng.choice([1.0, 2.0, 4.0, 8.0], size=n)
dev = torch.device("cuda", 0)
ctx = P.Context(0)
L = P.lib()
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
d_s = torch.from_numpy(s).to(dev)
out = {"n": n, "repeat": rep}
for name, tie in (("burst_ties", np.arange(n, dtype=np.uint32)),
                  ("shuffled_ties", rng.permutation(n).astype(np.uint32)),
                  ("no_ties", None)):
    d_t = torch.from_numpy(tie.astype(np.int32)).to(dev) if tie is not None else None
    d_o = torch.empty(n, dtype=torch.int32, device=dev)

    def run():
        assert L.pars_dev_priority_order(ctx.h, d_s.data_ptr(), None,
                                         d_t.data_ptr() if d_t is not None else None, n,
                                         d_o.data_ptr(), st.cuda_stream) == 0
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = 20
    a.record(st)
    for _ in range(k):
        run()
    b.record(st)
    torch.cuda.synchronize()
    out[name + "_ms"] = a.elapsed_time(b) / k
    # the same call captured once as a CUDA graph and replayed: device time
    # without the host's per-launch submission cost
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        run()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a.record(st)
    for _ in range(k):
        g.replay()
    b.record(st)
    torch.cuda.synchronize()
    out[name + "_graph_ms"] = a.elapsed_time(b) / k
    t = tie if tie is not None else np.zeros(n, np.uint32)
    ref = np.lexsort((np.arange(n), t, s))
    out[name + "_exact"] = bool((d_o.cpu().numpy() == ref).all())
print(json.dumps(out))
