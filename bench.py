"""Benchmark of the B200 PARS predictor hot path (BASELINE.json metric:
prompts scored/s, with filtered pairs/s and Kendall-tau reported beside it).

Workload (config C4 of BASELINE.json, the one the prompts-scored/s metric is
quoted on at 1/2/4/8 GPUs): 1,000,000 synthetic prompts from the reference
generator (synthesize_dataset seed 31) padded to 512 whitespace tokens with
" w<k>" filler; the reference's default predictor (hashed word
unigrams + char trigrams, D=4096, L2) with seeded random weights.
One step = score every prompt of the rank's shard (fused featurize + dot,
exact fp64 mode, bit-identical to the reference) and sort the shard into SJF
queue order (stable radix on (score, tie rank)). N GPUs split the 1M prompts
into contiguous shards (strong scaling, no data-path collective). Inputs
(2.1 GB of text) are larger than the 126 MB L2, so no flush is needed.

Secondary (same JSON line, key "pairs"): config C5 — the all-pairs
margin-ranking loss step over 65,536 prompts (Eq. 1 mask, hinge, integer
gradient coefficients): filtered pairs/s, tiles split across ranks.

Launch: python bench.py [--gpus N --steps K --warmup W] (torchrun for N>1).
        python bench.py --impl reference   -> the reference's CPU path
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_PROMPTS = 1_000_000
PAD_TOKENS = 512
SEED, PAD_SEED = 31, 5
C5_N, C5_SEED = 65536, 25
DELTA, MARGIN = 0.2, 1.0
DIM = 4096


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier_max(world, value):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def shard(n, world, rank):
    per = (n + world - 1) // world
    return min(n, rank * per), min(n, (rank + 1) * per)


def cpu_reference_scoring(wl, w, sample_n, threads):
    """The reference library (oracle/_ref, compiled from /root/reference) on
    the host cores: Scorer::score_batch (OpenMP) + select_batch over a
    bounded sample of the same workload."""
    from oracle.bind import Extractor as OEx
    from oracle.bind import Ref
    R = Ref()
    R.set_threads(threads)
    b, e = 0, sample_n
    offs = wl.offsets[b:e + 1] - wl.offsets[b]
    text = wl.text[wl.offsets[b]:wl.offsets[e]]
    ds = R.from_arrays(text, offs, wl.output_len[b:e], wl.prompt_len[b:e])
    ids = ["p%06d" % i for i in range(sample_n)]
    ex = OEx.make()
    R.score_batch(ex, ds, w)  # warm
    t0 = time.perf_counter()
    s = R.score_batch(ex, ds, w)
    t1 = time.perf_counter()
    R.select_batch(np.zeros(sample_n), ids, s, np.zeros(sample_n, np.uint8), 0.0, sample_n)
    t2 = time.perf_counter()
    return sample_n / (t2 - t0), (t1 - t0), (t2 - t1), s


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2510_03243_b200 import Workload
    # the reference's own generator would produce the identical text; ours is
    # pinned bit-identical to it (tests/test_abi.py) and much faster
    sample = args.cpu_sample
    wl = Workload.synthesize(sample, SEED, pad_tokens=PAD_TOKENS, pad_seed=PAD_SEED)
    w = np.random.default_rng(1234).normal(size=DIM) * 0.05
    threads = host_threads()
    vals = []
    for _ in range(args.warmup):
        cpu_reference_scoring(wl, w, sample, threads)
    for _ in range(args.steps):
        v, _, _, _ = cpu_reference_scoring(wl, w, sample, threads)
        vals.append(v)
    value = float(np.median(vals))
    line = {
        "impl": "reference", "metric": "prompts scored/s", "value": value, "unit": "prompts/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sample / value, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C4: score + SJF-sort 1M prompts x 512 tokens (reference CPU, "
                               f"bounded sample of {sample} prompts per step)",
                   "global_batch": N_PROMPTS, "seq_len": PAD_TOKENS, "parallelism": "openmp"},
        "cpu_baseline": {"value": value, "unit": "prompts/s", "cores": threads, "kind": "reference",
                         "sample": f"first {sample} prompts of the C4 workload, score_batch + select_batch"},
        "e2e": {"value": value, "unit": "prompts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def run_ours(args):
    import torch
    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2510_03243_b200 as P

    t_gen = time.perf_counter()
    wl = P.Workload.synthesize(N_PROMPTS, SEED, pad_tokens=PAD_TOKENS, pad_seed=PAD_SEED)
    t_gen = time.perf_counter() - t_gen
    b, e = shard(N_PROMPTS, world, rank)
    n = e - b
    t0b, t1b = int(wl.offsets[b]), int(wl.offsets[e])
    text_bytes = t1b - t0b
    w = np.random.default_rng(1234).normal(size=DIM) * 0.05
    ex = P.Extractor.make()
    ctx = P.Context(local)

    # device-resident inputs (torch owns the memory; the C ABI gets pointers)
    d_text = torch.from_numpy(wl.text[t0b:t1b]).to(dev)
    d_offs = torch.from_numpy(wl.offsets[b:e + 1] - t0b).to(dev)
    d_w = torch.from_numpy(w).to(dev)
    d_scores = torch.empty(n, dtype=torch.float64, device=dev)
    d_tie = torch.arange(b, e, dtype=torch.int32, device=dev)  # burst: rank of (0, id) = index
    d_order = torch.empty(n, dtype=torch.int32, device=dev)
    L = P.lib()
    # a dedicated (non-NULL) stream: a NULL handle would mean "the ctx's own
    # stream" to the C ABI and torch's events would not see the kernels
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        rc = L.pars_dev_score_text(ctx.h, __import__("ctypes").byref(ex), d_text.data_ptr(),
                                   d_offs.data_ptr(), n, d_w.data_ptr(), 0.0, P.MODE_EXACT,
                                   d_scores.data_ptr(), sh)
        if rc != 0:
            raise P.ParsError(rc, L.pars_last_error().decode())
        if ev is not None:
            ev[1].record(stream)
        rc = L.pars_dev_priority_order(ctx.h, d_scores.data_ptr(), None, d_tie.data_ptr(), n,
                                       d_order.data_ptr(), sh)
        if rc != 0:
            raise P.ParsError(rc, L.pars_last_error().decode())
        if ev is not None:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # parity spot check of this shard against the oracle (small sample, untimed)
    from oracle.bind import Extractor as OEx
    from oracle.bind import Oracle
    o = Oracle()
    chk = min(2000, n)
    so = o.score_batch(OEx.make(), wl.text, wl.offsets[b:b + chk + 1], w, 0.0)
    got = d_scores[:chk].cpu().numpy()
    parity_ok = bool((got.view(np.uint64) == so.view(np.uint64)).all())

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    launches0 = ctx.launches
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    start.record(stream)
    for k in range(args.steps):
        step(evs[k])
    stop.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier(world)
    launches = ctx.launches - launches0
    ms_local = start.elapsed_time(stop)
    ms = barrier_max(world, ms_local)
    ms_step = ms / args.steps
    value = N_PROMPTS / (ms_step / 1e3) if world > 1 else n / (ms_step / 1e3)
    feat_ms = float(np.mean([a.elapsed_time(b_) for a, b_, _ in evs]))
    sort_ms = float(np.mean([b_.elapsed_time(c) for _, b_, c in evs]))

    # roofline of the dominant kernel (fused featurize+score): algorithmic bytes
    alg_bytes = text_bytes + 8 * (n + 1) + 8 * n + 8 * DIM
    hbm, peak_kind = peaks()
    achieved = alg_bytes / (feat_ms / 1e3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / "featurize_ncu.json"
    if prof.exists():
        try:
            pj = json.loads(prof.read_text())
            traffic = pj.get("dram_bytes_per_launch_scaled")
        except Exception:
            traffic = None

    # e2e through the host-buffer C ABI (H2D text+offsets, D2H scores+order)
    ids_rank = np.arange(b, e, dtype=np.uint32)
    e2e_vals = []
    if n > 0 and not args.no_e2e:
        sub_offs = wl.offsets[b:e + 1]
        txt = wl.text  # pinned arena, offsets absolute
        for k in range(max(1, args.e2e_steps) + 1):
            barrier(world)
            t0 = time.perf_counter()
            s = ctx.score_text(ex, txt, sub_offs, w, 0.0, P.MODE_EXACT)
            order = ctx.priority_order(s, ids_rank)
            t1 = time.perf_counter()
            if k > 0:
                e2e_vals.append(barrier_max(world, t1 - t0))
    e2e_s = float(np.median(e2e_vals)) if e2e_vals else float("nan")
    e2e_vals_ok = bool(e2e_vals)
    e2e_value = (N_PROMPTS if world > 1 else n) / e2e_s
    h2d = text_bytes + 8 * (n + 1) + 8 * DIM + 4 * n
    d2h = 8 * n + 4 * n

    # secondary: C5 all-pairs step (filtered pairs/s)
    pairs = None
    if not args.no_pairs:
        pairs = bench_pairs(P, ctx, torch, dev, stream, world, rank, args)

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            thr = host_threads()
            v, ts, tsel, _ = cpu_reference_scoring(wl, w, args.cpu_sample, thr)
            cpu = {"value": v, "unit": "prompts/s", "cores": thr, "kind": "reference",
                   "sample": f"first {args.cpu_sample} prompts of the same C4 workload: "
                             f"score_batch ({ts:.2f} s, OpenMP {thr} threads) + select_batch ({tsel:.3f} s)"}
        line = {
            "metric": "prompts scored/s", "value": value, "unit": "prompts/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "C4: score + SJF-sort 1M synthetic prompts x 512 tokens "
                                   "(exact fp64 mode, bit-identical to the reference)",
                       "global_batch": N_PROMPTS, "seq_len": PAD_TOKENS,
                       "parallelism": f"shard{world}", "extractor": "hashed word{1}+char{3}, D=4096, L2",
                       "l2_flush": "inputs larger than L2 (%.2f GB text per rank)" % (text_bytes / 1e9)},
            "roofline": {"bound": "hbm", "kernel": "featurize_kernel (fused tokenise+hash+histogram+L2+dot)",
                         "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "peak_kind": peak_kind, "traffic": traffic,
                         "algorithmic_bytes_per_launch": alg_bytes, "kernel_ms": feat_ms,
                         "sort_ms": sort_ms},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "prompts/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "api": "pars_score_text + pars_priority_order (host buffers)"},
            "gpu_launches": int(launches),
            "clocks": clk,
            "parity": {"scores_bitexact_sample": parity_ok, "sample": chk},
            "pairs": pairs,
            "workload_gen_s": t_gen,
        }
        print(json.dumps(line))
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def bench_pairs(P, ctx, torch, dev, stream, world, rank, args):
    """C5: all-pairs loss step over 65,536 prompts, tiles split over ranks."""
    import ctypes as C
    wl = P.Workload.synthesize(C5_N, C5_SEED)
    w = np.random.default_rng(99).normal(size=DIM) * 0.05
    ex = P.Extractor.make()
    s = ctx.score_text(ex, wl.text, wl.offsets, w)
    lens = wl.output_len.astype(np.int32)
    max_len = int(lens.max())
    d_s = torch.from_numpy(s).to(dev)
    d_L = torch.from_numpy(lens).to(dev)
    from paper_2510_03243_b200 import distributed as D
    sh = stream.cuda_stream
    res = {}
    # per-dataset plan (lengths are fixed across steps): stable length order,
    # first kept column per row, exact kept count
    plan = ctx.pair_plan(wl.output_len, DELTA)

    def step():
        # this rank's tile slice on the GPU + NCCL all-reduce of the integer
        # coefficients/counters + tile-ordered loss reduction
        res["out"] = D.allpairs_step_gpu(ctx, d_s, d_L, C5_N, DELTA, MARGIN, max_len, stream=sh,
                                         plan=plan)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    barrier(world)
    a, bb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = max(3, args.steps)
    a.record(stream)
    for _ in range(k):
        step()
    bb.record(stream)
    torch.cuda.synchronize()
    ms = barrier_max(world, a.elapsed_time(bb)) / k
    _, kept, active, loss = res["out"]
    # exactness check against the golden exhaustive count
    return {"metric": "filtered pairs/s", "value": kept / (ms / 1e3), "unit": "pairs/s",
            "ms_per_step": ms, "kept": kept, "kept_expected": 1920977782, "active": active,
            "loss_sum": loss,
            "plan_sorted": plan.sorted,
            "workload": "C5: all 2,147,450,880 unordered pairs of 65,536 prompts (seed 25), "
                        "Eq.1 mask delta=0.2 + hinge + integer grad coefficients (fp64 scores)",
            "bound": "issue (int/fp64 ALU); inputs 0.5 MB are L2-resident"}


def main():
    global N_PROMPTS
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=20000)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-pairs", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--prompts", type=int, default=N_PROMPTS, help="(profiling only) fewer prompts")
    args = ap.parse_args()
    N_PROMPTS = args.prompts
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
