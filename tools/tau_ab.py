"""Timing + exactness of the sorted Kendall tau-b path (pars_dev_kendall_tau)
on the bench's workload shape: n random-normal scores against integer
output lengths (heavy ties in y), device-resident, CUDA events over
`reps` calls; counts checked against the all-pairs tile path.
  python tools/tau_ab.py [n] [reps]
Select an A/B build with PARS_CUDA_LIB=build_var/NAME/libpars_cuda.so."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_03243_b200 as P  # noqa: E402
from paper_2510_03243_b200 import distributed as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
rng = np.random.default_rng(11)
x = rng.normal(size=n)
y = np.floor(rng.lognormal(5.0, 1.0, size=n)).astype(np.float64)
dev = torch.device("cuda", 0)
ctx = P.Context(0)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
dx, dy = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
sh = st.cuda_stream
out = {"n": n, "reps": reps}
for _ in range(3):
    r = ctx.dev_kendall_tau(dx.data_ptr(), dy.data_ptr(), n, stream=sh)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(reps):
    r = ctx.dev_kendall_tau(dx.data_ptr(), dy.data_ptr(), n, stream=sh)
b.record(st)
torch.cuda.synchronize()
out["ms_per_call"] = a.elapsed_time(b) / reps
tau, c = r
tp, cp = D.kendall_tau_gpu(ctx, dx, dy, n, stream=sh)
out["tau_b"] = tau
out["counts_equal_pairs_path"] = [int(v) for v in c] == [int(v) for v in cp]
# graph replay over new contents of the same buffers, then a shorter n on
# the same pointers (re-capture): counts against the tile path each time
dx.copy_(torch.from_numpy(rng.normal(size=n)).to(dev))
t1, c1 = ctx.dev_kendall_tau(dx.data_ptr(), dy.data_ptr(), n, stream=sh)
t2, c2 = D.kendall_tau_gpu(ctx, dx, dy, n, stream=sh)
out["replay_new_contents_equal"] = [int(v) for v in c1] == [int(v) for v in c2]
h = n // 2 + 1
t1, c1 = ctx.dev_kendall_tau(dx.data_ptr(), dy.data_ptr(), h, stream=sh)
t2, c2 = D.kendall_tau_gpu(ctx, dx[:h].contiguous(), dy[:h].contiguous(), h, stream=sh)
out["recapture_shorter_equal"] = [int(v) for v in c1] == [int(v) for v in c2]
# non-finite inputs: the sorted path must step aside (same counts as tiles)
xn = x.copy()
xn[n // 3] = np.inf
dxn = torch.from_numpy(xn).to(dev)
t1, c1 = ctx.dev_kendall_tau(dxn.data_ptr(), dy.data_ptr(), n, stream=sh)
t2, c2 = D.kendall_tau_gpu(ctx, dxn, dy, n, stream=sh)
out["nonfinite_equal"] = [int(v) for v in c1] == [int(v) for v in c2]
print(json.dumps(out))
