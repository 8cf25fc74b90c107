"""Multi-GPU plumbing (one process per GPU, torch.distributed / NCCL).

Only the paths that shard naturally are partitioned:

* scoring: contiguous prompt ranges per rank, no data-path collective
  (`shard_range`, `score_shard`); an optional all-gather assembles the
  global score vector for a global SJF order;
* all-pairs loss (config C5): the upper-triangle tile list is split evenly
  across ranks (`tile_range`); each rank accumulates integer gradient
  coefficients, kept/active counts and per-tile loss partials; the exchange
  is an all-reduce of the int32 coefficients and int64 counters (exact for
  any rank count) and an all-gather of the per-tile partials, summed in tile
  order so the loss is bit-identical for 1, 2, 4 or 8 ranks;
* full-batch step: grad = X^T c over each rank's row shard, all-reduced
  (D doubles), then the update.

`kendall_tau_dp` splits kendall_tau_b's O(n^2) pair counts over the same
upper-triangle tiles; the exchange is one all-reduce of 4 integer counts.

`train_step` is the whole C5 data-parallel step — score this rank's prompt
shard with the current weights, all-gather the scores, the rank's all-pairs
tiles, the coefficient all-reduce, X^T c on the row shard, the gradient
all-reduce and w -= (lr / kept) * grad — with every collective on device
tensors and no host synchronisation inside the step.

The per-rank compute is the CUDA kernel (`pars_dev_allpairs`); the CPU tests
substitute a reference implementation of the same per-tile contract to check
the partition and the collectives with the gloo backend.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional, Tuple

import numpy as np

TILE = 256  # pairs.cu kTile


def shard_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    per = (n + world - 1) // world
    return min(n, rank * per), min(n, (rank + 1) * per)


def tile_count(n: int) -> int:
    nt = (n + TILE - 1) // TILE
    return nt * (nt + 1) // 2


def tile_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Equal share of the upper-triangle tile list (tiles are equal-cost
    except the diagonal ones, which are half-empty)."""
    return shard_range(tile_count(n), world, rank)


def tile_coords(t: int, n: int) -> Tuple[int, int]:
    """Row-major upper-triangle enumeration (pairs.cu tile_of)."""
    nt = (n + TILE - 1) // TILE
    i = 0
    while i + 1 < nt and (i + 1) * nt - (i + 1) * i // 2 <= t:
        i += 1
    start = i * nt - i * (i - 1) // 2
    return i, i + (t - start)


def _dist():
    import torch.distributed as dist
    return dist


def _gpu_tiles(ctx, d_scores, d_lengths, n, delta, margin, max_len, stream, plan=None):
    """Per-rank compute on the GPU for tiles [t0, t1): the length-sorted
    kernel when a PairPlan is given, else the general tiled kernel."""
    import torch
    from ._lib import ParsError, lib

    def run(t0: int, t1: int, scores=None):
        d_s = d_scores if scores is None else scores
        dev = d_s.device
        c = torch.zeros(n, dtype=torch.int32, device=dev)
        cnt = torch.zeros(4, dtype=torch.int64, device=dev)
        part = torch.zeros(max(1, t1 - t0), dtype=torch.float64, device=dev)
        if plan is not None:
            plan.run(d_s.data_ptr(), margin, t0, t1, c.data_ptr(), cnt.data_ptr(),
                     part.data_ptr(), stream or 0)
        else:
            rc = lib().pars_dev_allpairs(ctx.h, d_s.data_ptr(), d_lengths.data_ptr(), n, delta,
                                         margin, max_len, t0, t1, c.data_ptr(), cnt.data_ptr(),
                                         part.data_ptr(), stream)
            if rc != 0:
                raise ParsError(rc, lib().pars_last_error().decode("utf-8", "replace"))
        return c, cnt[:2], part[: max(0, t1 - t0)]

    return run


def allpairs_dp(n: int, compute: Callable, group=None):
    """All-pairs margin-ranking loss over n prompts split across the ranks of
    `group` (or a single process when torch.distributed is not initialised).

    compute(t0, t1) -> (coeff int32[n], counts int64[2] = kept, active,
    loss partials float64[t1-t0]) for this rank's tile slice.
    Returns (coeff, kept, active, loss_sum) identical on every rank."""
    import torch
    dist = _dist()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    t0, t1 = tile_range(n, world, rank)
    c, cnt, part = compute(t0, t1)
    if world > 1:
        dist.all_reduce(c, group=group)
        dist.all_reduce(cnt, group=group)
        # per-tile partials, gathered into tile order, then one fixed-order sum
        sizes = [tile_range(n, world, r) for r in range(world)]
        width = max(b - a for a, b in sizes)
        buf = torch.zeros(width, dtype=torch.float64, device=part.device)
        buf[: part.numel()] = part
        bufs = [torch.zeros_like(buf) for _ in range(world)]
        dist.all_gather(bufs, buf, group=group)
        part = torch.cat([bufs[r][: sizes[r][1] - sizes[r][0]] for r in range(world)])
    loss = float(part.sum().item()) if part.numel() else 0.0
    return c, int(cnt[0].item()), int(cnt[1].item()), loss


def allpairs_step_gpu(ctx, d_scores, d_lengths, n: int, delta: float, margin: float, max_len: int,
                      stream: int = 0, group=None, plan=None):
    """The C5 exchange step on GPUs (NCCL when the group is initialised).
    `plan` (Context.pair_plan(lengths, delta)) selects the length-sorted kernel."""
    return allpairs_dp(n, _gpu_tiles(ctx, d_scores, d_lengths, n, delta, margin, max_len,
                                     stream or None, plan), group)


def grad_step_gpu(ctx, feats, d_coeff, scale: float, group=None, stream: int = 0):
    """grad = scale * X^T c over this rank's row shard, all-reduced."""
    import torch
    from ._lib import ParsError, lib
    dist = _dist()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    r0, r1 = shard_range(feats.rows, world, rank)
    g = torch.zeros(feats.dim, dtype=torch.float64, device=d_coeff.device)
    rc = lib().pars_dev_xt_c(ctx.h, C.c_void_p(feats.h), d_coeff.data_ptr(), r0, r1, g.data_ptr(),
                             stream or None)
    if rc != 0:
        raise ParsError(rc, lib().pars_last_error().decode("utf-8", "replace"))
    if world > 1:
        dist.all_reduce(g, group=group)
    return g * scale


def train_step(n: int, w, scores_pad, score_rows: Callable, tiles: Callable, xt_c: Callable,
               lr_over_kept: float, group=None):
    """One full-batch data-parallel step of all-pairs margin-ranking training.

    w             device float64[D], updated in place
    scores_pad    device float64[per * world] (per = ceil(n / world)); rank r
                  owns [r*per, r*per + shard); the first n entries end up as
                  the full score vector on every rank
    score_rows(r0, r1, out)  writes scores of prompts [r0, r1) into out[0:r1-r0]
    tiles(scores, t0, t1)    -> (coeff int32[n], counts int64[2], loss partials)
    xt_c(coeff, r0, r1)      -> float64[D] = X[r0:r1]^T coeff[r0:r1]
    Returns device tensors (counts = kept, active; loss partials of this
    rank's tiles, in tile order)."""
    dist = _dist()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    per = (n + world - 1) // world
    r0, r1 = shard_range(n, world, rank)
    mine = scores_pad[rank * per:(rank + 1) * per]
    if r1 > r0:
        score_rows(r0, r1, mine)
    if world > 1:
        dist.all_gather_into_tensor(scores_pad, mine, group=group)
    t0, t1 = tile_range(n, world, rank)
    c, cnt, part = tiles(scores_pad[:n], t0, t1)
    if world > 1:
        dist.all_reduce(c, group=group)
        dist.all_reduce(cnt, group=group)
    g = xt_c(c, r0, r1)
    if world > 1:
        dist.all_reduce(g, group=group)
    w.sub_(g * lr_over_kept)
    return cnt, part


def train_step_gpu(ctx, feats, d_w, scores_pad, d_lengths, n: int, delta: float, margin: float,
                   max_len: int, lr_over_kept: float, stream: int = 0, group=None, plan=None):
    """train_step with the CUDA kernels: pars_dev_features_score (exact CSR
    dot), the all-pairs tiles (length-sorted plan kernel when `plan` is
    given) and pars_dev_xt_c."""
    import torch
    from ._lib import ParsError, lib

    def check(rc):
        if rc != 0:
            raise ParsError(rc, lib().pars_last_error().decode("utf-8", "replace"))

    def score_rows(r0, r1, out):
        # the kernel writes d_scores[r0:r1]; point it so that lands in out
        base = out.data_ptr() - r0 * 8
        check(lib().pars_dev_features_score(ctx.h, C.c_void_p(feats.h), r0, r1, d_w.data_ptr(),
                                            0.0, base, stream or None))

    gpu_tiles = _gpu_tiles(ctx, None, d_lengths, n, delta, margin, max_len, stream or None, plan)

    def tiles(scores, t0, t1):
        return gpu_tiles(t0, t1, scores)

    def xt_c(c, r0, r1):
        g = torch.empty(feats.dim, dtype=torch.float64, device=d_w.device)
        check(lib().pars_dev_xt_c(ctx.h, C.c_void_p(feats.h), c.data_ptr(), r0, r1, g.data_ptr(),
                                  stream or None))
        return g

    return train_step(n, d_w, scores_pad, score_rows, tiles, xt_c, lr_over_kept, group)


def kendall_tau_dp(n: int, counts: Callable, finish: Callable, group=None):
    """kendall_tau_b (metrics.cpp:42-64) over n items with the pair tiles split
    across ranks: counts(t0, t1) -> int64[4] {n_c, n_d, n1, n2} of this rank's
    tiles; one exact all-reduce; finish(totals) -> (tau_b, counts5)."""
    dist = _dist()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    t0, t1 = tile_range(n, world, rank)
    c = counts(t0, t1)
    if world > 1:
        dist.all_reduce(c, group=group)
    return finish(c)


def kendall_tau_gpu(ctx, d_x, d_y, n: int, stream: int = 0, group=None):
    """kendall_tau_dp with the CUDA tile kernel (pars_dev_kendall_counts) and
    the reference's finish_tau (pars_kendall_finish)."""
    import numpy as np
    import torch
    from ._lib import ParsError, lib

    def counts(t0, t1):
        c = torch.zeros(4, dtype=torch.int64, device=d_x.device)
        rc = lib().pars_dev_kendall_counts(ctx.h, d_x.data_ptr(), d_y.data_ptr(), n, t0, t1,
                                           c.data_ptr(), stream or None)
        if rc != 0:
            raise ParsError(rc, lib().pars_last_error().decode("utf-8", "replace"))
        return c

    def finish(c):
        c4 = np.ascontiguousarray(c.cpu().numpy().astype(np.uint64))
        c5 = np.zeros(5, np.uint64)
        tau = C.c_double()
        rc = lib().pars_kendall_finish(c4.ctypes.data, n, c5.ctypes.data, C.byref(tau))
        if rc != 0:
            raise ParsError(rc, lib().pars_last_error().decode("utf-8", "replace"))
        return tau.value, c5

    return kendall_tau_dp(n, counts, finish, group)
