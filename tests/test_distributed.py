"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU plumbing:
tile partition, coefficient/counter all-reduce and the fixed-order loss
reduction. The per-rank compute is a numpy restatement of the all-pairs
tile contract (pairs.cu), checked against the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_03243_b200 import distributed as D


def rel(a, b):
    return abs(a - b) / max(a, b)


def tile_compute_numpy(s, lens, delta, margin):
    """Per-rank compute with the kernel's contract for tiles [t0, t1)."""
    n = len(s)

    def run(t0, t1):
        c = np.zeros(n, np.int64)
        kept = act = 0
        parts = []
        for t in range(t0, t1):
            I, J = D.tile_coords(t, n)
            loss = 0.0
            for i in range(I * D.TILE, min(n, (I + 1) * D.TILE)):
                for j in range(J * D.TILE, min(n, (J + 1) * D.TILE)):
                    if I == J and j <= i:
                        continue
                    la, lb = int(lens[i]), int(lens[j])
                    if la == lb or rel(la, lb) < delta:
                        continue
                    kept += 1
                    y = 1 if la > lb else -1
                    h = -y * (s[i] - s[j]) + margin
                    if h > 0:
                        act += 1
                        loss += h
                        c[i] -= y
                        c[j] += y
            parts.append(loss)
        return (torch.tensor(c, dtype=torch.int32), torch.tensor([kept, act], dtype=torch.int64),
                torch.tensor(parts, dtype=torch.float64))

    return run


def test_tile_partition_covers_every_tile_once():
    for n in (1, 2, 255, 256, 257, 700, 2049):
        T = D.tile_count(n)
        for world in (1, 2, 3, 4, 8):
            got = []
            for r in range(world):
                a, b = D.tile_range(n, world, r)
                got.extend(range(a, b))
            assert got == list(range(T))
        nt = (n + D.TILE - 1) // D.TILE
        coords = [D.tile_coords(t, n) for t in range(T)]
        assert coords == [(i, j) for i in range(nt) for j in range(i, nt)]


def test_shard_range_covers_prompts():
    for n in (0, 1, 7, 1000):
        for world in (1, 2, 4, 8):
            idx = []
            for r in range(world):
                a, b = D.shard_range(n, world, r)
                idx.extend(range(a, b))
            assert idx == list(range(n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, s, lens, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c, kept, act, loss = D.allpairs_dp(len(s), tile_compute_numpy(s, lens, 0.2, 1.0))
        out[rank] = (c.numpy().tolist(), kept, act, loss)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_allpairs_dp_gloo_matches_single_process_and_oracle(world, oracle):
    rng = np.random.default_rng(5)
    n = 600
    lens = rng.integers(1, 300, size=n)
    s = rng.normal(size=n)
    single = D.allpairs_dp(n, tile_compute_numpy(s, lens, 0.2, 1.0))
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, s, lens, out), nprocs=world, join=True,
                       start_method="fork")
    oc, okept, oact, oloss = oracle.allpairs(s, lens, 0.2, 1.0)
    for r in range(world):
        c, kept, act, loss = out[r]
        assert c == oc.tolist() and kept == okept and act == oact
        assert c == single[0].numpy().tolist() and kept == single[1] and act == single[2]
        # per-tile partials summed in tile order: bit-identical for any world size
        assert loss == single[3]
        assert abs(loss - oloss) <= 1e-12 * max(1.0, oloss)


def _step_fns(X, lens, delta, margin):
    """CPU stand-ins for the three per-rank kernels of train_step."""
    def score_rows(r0, r1, out):
        out[: r1 - r0] = torch.from_numpy(X[r0:r1]) @ W["w"]

    def tiles(scores, t0, t1):
        return tile_compute_numpy(scores.numpy(), lens, delta, margin)(t0, t1)

    def xt_c(c, r0, r1):
        return torch.from_numpy(X[r0:r1].T) @ c[r0:r1].to(torch.float64)

    return score_rows, tiles, xt_c


W = {}


def _step_worker(rank, world, port, X, lens, w0, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = X.shape[0]
        w = torch.tensor(w0)
        W["w"] = w
        per = (n + world - 1) // world
        pad = torch.zeros(per * world, dtype=torch.float64)
        fns = _step_fns(X, lens, 0.2, 1.0)
        cnt, _ = D.train_step(n, w, pad, *fns, lr_over_kept=0.1 / 1000)
        out[rank] = (w.numpy().tolist(), cnt.numpy().tolist(), pad[:n].numpy().tolist())
    finally:
        dist.destroy_process_group()


def test_train_step_gloo_matches_single_process():
    """The full DP step (shard scoring + score all-gather, tile slice +
    coefficient all-reduce, X^T c + gradient all-reduce, update) on 2 ranks
    equals the single-process step: scores and integer counts exactly, the
    weights to fp64 summation-order rounding."""
    rng = np.random.default_rng(9)
    n, dim = 300, 16
    X = rng.normal(size=(n, dim))
    lens = rng.integers(1, 200, size=n)
    w0 = rng.normal(size=dim) * 0.1
    w1 = torch.tensor(w0)
    W["w"] = w1
    pad = torch.zeros(n, dtype=torch.float64)
    cnt1, _ = D.train_step(n, w1, pad, *_step_fns(X, lens, 0.2, 1.0), lr_over_kept=0.1 / 1000)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_step_worker, args=(2, _free_port(), X, lens, w0, out), nprocs=2, join=True,
                       start_method="fork")
    for r in range(2):
        w, cnt, sc = out[r]
        assert cnt == cnt1.numpy().tolist()
        np.testing.assert_allclose(sc, X @ w0, rtol=1e-13, atol=1e-14)
        np.testing.assert_allclose(w, w1.numpy(), rtol=1e-12, atol=1e-15)


def _tau_counts_numpy(x, y):
    """Per-tile Kendall counts with the kernel's contract (pairs.cu tau_kernel)."""
    n = len(x)

    def run(t0, t1):
        nc = nd = n1 = n2 = 0
        for t in range(t0, t1):
            I, J = D.tile_coords(t, n)
            for i in range(I * D.TILE, min(n, (I + 1) * D.TILE)):
                for j in range(J * D.TILE, min(n, (J + 1) * D.TILE)):
                    if I == J and j <= i:
                        continue
                    dx, dy = x[i] - x[j], y[i] - y[j]
                    n1 += dx == 0
                    n2 += dy == 0
                    if dx != 0 and dy != 0:
                        if (dx > 0) == (dy > 0):
                            nc += 1
                        else:
                            nd += 1
        return torch.tensor([nc, nd, n1, n2], dtype=torch.int64)

    return run


def _tau_worker(rank, world, port, x, y, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = D.kendall_tau_dp(len(x), _tau_counts_numpy(x, y), lambda t: t.numpy().tolist())
        out[rank] = c
    finally:
        dist.destroy_process_group()


def test_kendall_tau_dp_gloo_matches_oracle(oracle):
    """Tiles split over 2 ranks + one integer all-reduce = the reference's
    counts (oracle kendall)."""
    rng = np.random.default_rng(4)
    n = 520
    x = rng.integers(0, 40, n).astype(np.float64)
    y = rng.integers(0, 30, n).astype(np.float64)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_tau_worker, args=(2, _free_port(), x, y, out), nprocs=2, join=True,
                       start_method="fork")
    single = D.kendall_tau_dp(n, _tau_counts_numpy(x, y), lambda t: t.numpy().tolist())
    assert out[0] == out[1] == single
    tau, counts = oracle.kendall(x, y)
    assert single == [int(counts[0]), int(counts[1]), int(counts[3]), int(counts[4])]
