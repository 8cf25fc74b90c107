"""The NCCL data-parallel layer of the C ABI (pars_dp_*).

CPU tests cover the host-only pieces (shard ranges, the cost-balanced split).
GPU tests run a world-1 NCCL communicator end to end (the only multi-GPU
configuration a one-GPU box can host) and check the pieces that make N > 1
correct on one device: every run placed separately by pars_dev_merge_rank
reproduces the full sort, and the per-rank tile slices of
pars_pair_plan_tile_split sum to the full all-pairs result."""
import numpy as np
import pytest

import paper_2510_03243_b200 as P
from paper_2510_03243_b200 import distributed as D


# ---- host-only ---------------------------------------------------------------

def test_dp_shard_matches_python_shards():
    for n in (0, 1, 7, 1000, 65536, 1000001):
        for world in (1, 2, 3, 4, 8):
            got = [P.dp_shard(n, world, r) for r in range(world)]
            assert got == [D.shard_range(n, world, r) for r in range(world)]


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_split_weighted_is_a_balanced_partition(world):
    rng = np.random.default_rng(world)
    for n in (0, 1, 5, 100, 32896):
        w = rng.choice([1, 64], size=n, p=[0.3, 0.7]).astype(np.int64)
        b = P.split_weighted(w, world)
        assert b[0] == 0 and b[-1] == n and (np.diff(b) >= 0).all()
        if n:
            per = [int(w[b[r]:b[r + 1]].sum()) for r in range(world)]
            # each rank within one item of its equal share
            assert max(abs(p - w.sum() / world) for p in per) <= w.max() + 1e-9


def test_split_weighted_rejects_bad_input():
    with pytest.raises(P.ParsError):
        P.split_weighted(np.array([1, -1, 2]), 2)
    with pytest.raises(P.ParsError):
        P.split_weighted(np.array([1, 2]), 0)


# ---- GPU -----------------------------------------------------------------

@pytest.fixture
def tstream():
    """A non-default torch stream made current for the test: the C ABI runs
    on it too, so torch's ops and the library's kernels are stream-ordered
    (a NULL handle would mean the ctx's own non-blocking stream)."""
    import torch
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        yield st.cuda_stream
    torch.cuda.synchronize()


def _dp1(ctx):
    import torch  # noqa: F401  (loads the process's libnccl, reused by the dp layer)
    return P.DataParallel(ctx, P.nccl_unique_id(), 1, 0)


@pytest.mark.gpu
@pytest.mark.parametrize("nruns", [1, 2, 3, 5, 8])
def test_merge_rank_places_each_run(ctx, nruns, tstream):
    """Runs placed one at a time (as data-parallel ranks do) into a zeroed
    order and summed equal one sort of everything."""
    import torch
    rng = np.random.default_rng(nruns)
    n = 20011
    s = np.round(rng.normal(size=n), 2)  # many equal scores
    s[::97] = -0.0
    boosted = (rng.random(n) < 0.05).astype(np.uint8)
    tie = rng.permutation(n).astype(np.uint32) // 3  # shared tie ranks too
    dev = torch.device("cuda", 0)
    d_s = torch.from_numpy(s).to(dev)
    d_b = torch.from_numpy(boosted).to(dev)
    d_t = torch.from_numpy(tie.astype(np.int32)).to(dev)
    off = np.array([n * r // nruns for r in range(nruns + 1)], np.int64)
    runs = torch.zeros(n, dtype=torch.int32, device=dev)
    L = P.lib()
    st = tstream
    for r in range(nruns):
        a, b = int(off[r]), int(off[r + 1])
        assert L.pars_dev_priority_order(ctx.h, d_s[a:].data_ptr(), d_b[a:].data_ptr(),
                                         d_t[a:].data_ptr(), b - a, runs[a:].data_ptr(), st) == 0
    total = torch.zeros(n, dtype=torch.int64, device=dev)
    for r in range(nruns):
        o = torch.zeros(n, dtype=torch.int32, device=dev)
        assert L.pars_dev_merge_rank(ctx.h, d_s.data_ptr(), d_b.data_ptr(), d_t.data_ptr(),
                                     runs.data_ptr(), off.ctypes.data, nruns, r, o.data_ptr(),
                                     st) == 0
        total += o.to(torch.int64)
    full = ctx.priority_order(s, tie, boosted)
    torch.cuda.synchronize()
    assert (total.cpu().numpy() == full).all()


@pytest.mark.gpu
def test_dp_world1_score_order_equals_single_gpu(ctx, tstream):
    import torch
    wl = P.Workload.synthesize(3000, 22, pad_tokens=64)
    ex = P.Extractor.make()
    w = np.random.default_rng(0).normal(size=4096) * 0.05
    dev = torch.device("cuda", 0)
    d_text = torch.from_numpy(wl.text[wl.offsets[0]:wl.offsets[-1]].copy()).to(dev)
    d_offs = torch.from_numpy(wl.offsets - wl.offsets[0]).to(dev)
    d_w = torch.from_numpy(w).to(dev)
    n = len(wl)
    tie = np.arange(n, dtype=np.uint32)[::-1].copy()  # non-trivial tie ranks
    d_tie = torch.from_numpy(tie.astype(np.int32)).to(dev)
    d_s = torch.empty(n, dtype=torch.float64, device=dev)
    d_o = torch.empty(n, dtype=torch.int32, device=dev)
    dp = _dp1(ctx)
    assert dp.world == 1 and dp.rank == 0
    dp.score_order(ex, d_text.data_ptr(), d_offs.data_ptr(), n, d_w.data_ptr(), 0.0, P.MODE_EXACT,
                   d_s.data_ptr(), d_o.data_ptr(), d_tie_all=d_tie.data_ptr(),
                   stream=tstream)
    torch.cuda.synchronize()
    s = ctx.score_text(ex, wl.text, wl.offsets, w, 0.0, P.MODE_EXACT)
    assert (d_s.cpu().numpy().view(np.uint64) == s.view(np.uint64)).all()
    assert (d_o.cpu().numpy() == ctx.priority_order(s, tie)).all()
    dp.close()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_tile_split_slices_sum_to_full(ctx, world, tstream):
    """The cost-balanced rank slices of the pair tiles cover every tile once:
    their integer coefficients and counts add up to the single-GPU result."""
    import torch
    wl = P.Workload.synthesize(5000, 25)
    plan = ctx.pair_plan(wl.output_len, 0.2)
    b = plan.tile_split(world)
    assert b[0] == 0 and b[-1] == P.lib().pars_allpairs_tiles(len(wl)) and (np.diff(b) >= 0).all()
    s = np.random.default_rng(1).normal(size=len(wl))
    dev = torch.device("cuda", 0)
    d_s = torch.from_numpy(s).to(dev)
    c = torch.zeros(len(wl), dtype=torch.int32, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    for r in range(world):
        part = torch.zeros(max(1, int(b[r + 1] - b[r])), dtype=torch.float64, device=dev)
        plan.run(d_s.data_ptr(), 1.0, int(b[r]), int(b[r + 1]), c.data_ptr(), cnt.data_ptr(),
                 part.data_ptr(), tstream)
    fc, fk, fa, _ = ctx.allpairs(s, wl.output_len, 0.2, 1.0)
    torch.cuda.synchronize()
    assert (c.cpu().numpy() == fc).all()
    assert int(cnt[0]) == fk == plan.kept and int(cnt[1]) == fa


@pytest.mark.gpu
def test_dp_world1_train_step_matches_oracle(ctx, oracle, tstream):
    """One full-batch step from w0: scores bit-exact, integer coefficients and
    counts bit-exact, the loss to 1e-12 relative, the updated weights to
    1e-12 of the step's magnitude (X^T c summed in a different order)."""
    import torch
    wl = P.Workload.synthesize(4096, 25)
    ex = P.Extractor.make()
    f = ctx.extract(ex, wl.text, wl.offsets)
    plan = ctx.pair_plan(wl.output_len, 0.2)
    w0 = np.random.default_rng(3).normal(size=4096) * 0.05
    dev = torch.device("cuda", 0)
    d_w = torch.from_numpy(w0.copy()).to(dev)
    n = len(wl)
    d_s = torch.empty(n, dtype=torch.float64, device=dev)
    d_c = torch.empty(n, dtype=torch.int32, device=dev)
    d_cnt = torch.empty(2, dtype=torch.int64, device=dev)
    d_loss = torch.empty(1, dtype=torch.float64, device=dev)
    dp = _dp1(ctx)
    lr, margin = 0.1, 1.0
    dp.train_step(f, plan, d_w.data_ptr(), margin, lr, d_c.data_ptr(), d_s.data_ptr(),
                  d_cnt.data_ptr(), d_loss.data_ptr(), stream=tstream)
    torch.cuda.synchronize()
    rp, idx, val = f.download()
    so = oracle.score_batch(P.Extractor.make(), wl.text, wl.offsets, w0, 0.0)
    assert (d_s.cpu().numpy().view(np.uint64) == so.view(np.uint64)).all()
    oc, okept, oact, oloss = oracle.allpairs(so, wl.output_len, 0.2, margin)
    assert (d_c.cpu().numpy() == oc).all()
    assert int(d_cnt[0]) == okept == plan.kept and int(d_cnt[1]) == oact
    assert abs(float(d_loss[0]) - oloss) <= 1e-12 * abs(oloss)
    g = oracle.xt_c(rp, idx, val, oc, 4096)
    mag = np.zeros(4096)
    rows = np.repeat(np.arange(n), np.diff(rp))
    np.add.at(mag, idx, np.abs(val * oc[rows]))
    w1 = w0 - (lr / okept) * g
    got = d_w.cpu().numpy()
    assert (np.abs(got - w1) <= 1e-12 * (lr / okept) * mag + 1e-300).all()
    dp.close()
    plan.free()
    f.free()


@pytest.mark.gpu
def test_dp_world1_kendall(ctx, tstream):
    import torch
    rng = np.random.default_rng(7)
    x = np.round(rng.normal(size=3001), 1)
    y = np.round(x + rng.normal(size=3001), 1)
    dev = torch.device("cuda", 0)
    d_x, d_y = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
    dp = _dp1(ctx)
    tau, counts = dp.kendall_tau(d_x.data_ptr(), d_y.data_ptr(), len(x),
                                 stream=tstream)
    t2, c2 = ctx.kendall_tau(x, y)
    assert tau == t2 and (counts == c2).all()
    dp.close()
