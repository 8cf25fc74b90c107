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
import hashlib
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
    """SM clock + throttle reasons DURING the timed region, polled through
    NVML every 2 ms on a background thread (nvidia-smi's start-up alone
    outlasts a short timed region); falls back to one nvidia-smi reading."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        self.device = device
        self.samples, self.mask, self.smax = [], 0, None
        self.stop_ev = threading.Event()
        self.nvml = None

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.device)
            self.smax = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            self.nvml = (N, h)
        except Exception:
            self.nvml = None
            return

        def poll():
            N, h = self.nvml
            get_reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
            while not self.stop_ev.is_set():
                try:
                    self.samples.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
                    self.mask |= int(get_reasons(h))
                except Exception:
                    pass
                time.sleep(0.002)

        self.t = threading.Thread(target=poll, daemon=True)
        self.t.start()

    def stop(self):
        if self.nvml is None:
            return self._smi_once()
        self.stop_ev.set()
        self.t.join(timeout=2)
        reasons = sorted(v for k, v in self.REASONS.items() if self.mask & k)
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.smax, "reasons": reasons, "samples": len(self.samples),
                "source": "NVML, 2 ms polling during the timed region"}

    def _smi_once(self):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                  "--query-gpu=clocks.sm,clocks.max.sm", "--format=csv,noheader,nounits"],
                                 capture_output=True, text=True, timeout=10).stdout.split(",")
            return {"sm_mhz": float(out[0]), "sm_max_mhz": float(out[1]), "reasons": [],
                    "samples": 1, "source": "nvidia-smi after the timed region"}
        except Exception:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock query unavailable"]}


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("PARS_DIST_BACKEND", "nccl") != "nccl":
        import torch
        local = local % max(1, torch.cuda.device_count())
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        # PARS_DIST_BACKEND=gloo: exercise the N>1 path with several ranks on
        # one GPU (NCCL refuses duplicate devices); the timed runs use NCCL
        backend = os.environ.get("PARS_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
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


class CpuReferenceScoring:
    """The reference library (oracle/_ref, compiled from /root/reference) on
    the host cores: Scorer::score_batch (OpenMP, all threads) + select_batch
    (ref_capi.cpp ref_score_order) over a bounded sample of the same
    workload."""

    def __init__(self, wl, w, sample_n, threads):
        from oracle.bind import Extractor as OEx
        from oracle.bind import Ref
        self.R = R = Ref()
        R.set_threads(threads)
        self.n = n = min(sample_n, len(wl))
        offs = wl.offsets[: n + 1] - wl.offsets[0]
        text = wl.text[wl.offsets[0]:wl.offsets[n]]
        self.ds = R.from_arrays(text, offs, wl.output_len[:n], wl.prompt_len[:n])
        self.ex = OEx.make()
        self.w = w

    def step(self):
        t0 = time.perf_counter()
        self.R.score_order(self.ex, self.ds, self.w)
        return self.n / (time.perf_counter() - t0)


def repo_native_loaded():
    """Shared objects of this repository mapped into this process (evidence of
    which native code ran: the product, the reference build, the tools)."""
    out = set()
    try:
        for ln in open("/proc/self/maps"):
            path = ln.split()[-1] if ln.strip() else ""
            if path.endswith(".so") and path.startswith(str(ROOT)):
                out.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(out)


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args):
    """The reference's own CPU path on this host, clean: only oracle/_ref (the
    reference library compiled from /root/reference, shipped prebuilt) and
    numpy are loaded — no module or shared object of this repository's
    product. Inputs come from the reference's own synthesize_dataset (seed 31)
    padded to 512 tokens by the reference's Rng (ref_capi.cpp ref_pad_dataset),
    i.e. the same 1M-prompt C4 workload as our arm (our generator is pinned
    bit-identical to it). One step = Scorer::score_batch over all 1M prompts
    (OpenMP, every host thread) + select_batch of the burst, the reference's
    stock code path (ref_capi.cpp ref_score_order)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.bind import Dataset as RefDataset
    from oracle.bind import Extractor as OEx
    from oracle.bind import Ref
    R = Ref()
    threads = host_threads()
    R.set_threads(threads)
    n = N_PROMPTS
    t0 = time.perf_counter()
    ds = RefDataset(R, R.L.ref_synthesize(n, 5.0, 1.2, SEED, 0, 0), export=False)
    R.pad_dataset(ds, PAD_TOKENS, PAD_SEED)
    t_gen = time.perf_counter() - t0
    w = np.random.default_rng(1234).normal(size=DIM) * 0.05
    ex = OEx.make()
    for _ in range(args.warmup):
        R.score_order(ex, ds, w)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        s, order = R.score_order(ex, ds, w)
        ts.append(time.perf_counter() - t0)
    step_s = float(np.median(ts))
    value = n / step_s
    line = {
        "impl": "reference", "metric": "prompts scored/s", "value": value, "unit": "prompts/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * step_s, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C4: score + SJF-sort 1M synthetic prompts x 512 tokens "
                               "(reference CPU: Scorer::score_batch + select_batch)",
                   "global_batch": n, "seq_len": PAD_TOKENS, "parallelism": "openmp",
                   "extractor": "hashed word{1}+char{3}, D=4096, L2",
                   "inputs": f"reference synthesize_dataset({n}, seed 31) + C4 padding (Rng seed 5)"},
        "cpu_baseline": {"value": value, "unit": "prompts/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"the full C4 workload ({n} prompts) per step; median of "
                                   f"{args.steps} steps"},
        "e2e": {"value": value, "unit": "prompts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        # digests of the last step's outputs, comparable with our arm's
        "outputs": {"scores_sha256": hashlib.sha256(s.tobytes()).hexdigest()[:32],
                    "order_sha256": hashlib.sha256(order.astype(np.int64).tobytes()).hexdigest()[:32]},
        "workload_gen_s": t_gen,
        "native_loaded": repo_native_loaded(),
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
    # shard buffers are `per` long (equal across ranks) so the all-gather of
    # the global-order step needs no padding logic; this rank fills the first n
    per = (N_PROMPTS + world - 1) // world
    d_scores = torch.empty(per, dtype=torch.float64, device=dev)
    d_tie = torch.arange(b, e, dtype=torch.int32, device=dev)  # burst: rank of (0, id) = index
    d_order = torch.zeros(per, dtype=torch.int32, device=dev)
    L = P.lib()
    # a dedicated (non-NULL) stream: a NULL handle would mean "the ctx's own
    # stream" to the C ABI and torch's events would not see the kernels
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream
    dp = make_dp(P, ctx, world, rank)
    if world > 1:
        # the global SJF order of all N prompts: every rank
        # ends with all N scores and the global order
        g_scores = torch.empty(N_PROMPTS, dtype=torch.float64, device=dev)
        g_order = torch.empty(N_PROMPTS, dtype=torch.int32, device=dev)
        g_tie = torch.arange(N_PROMPTS, dtype=torch.int32, device=dev)
        if dp is None:  # gloo test mode: gather through torch, merge on rank 0
            import torch.distributed as dist
            g_pad = torch.empty(per * world, dtype=torch.float64, device=dev)
            g_orders = torch.empty(per * world, dtype=torch.int32, device=dev)
            run_offs = np.array([min(N_PROMPTS, r * per) for r in range(world + 1)], np.int64)

            def gather_into(out, inp):
                parts = [torch.empty_like(inp, device="cpu") for _ in range(world)]
                dist.all_gather(parts, inp.cpu())
                out.copy_(torch.cat(parts))

    def check(rc):
        if rc != 0:
            raise P.ParsError(rc, L.pars_last_error().decode("utf-8", "replace"))

    def score_shard():
        check(L.pars_dev_score_text(ctx.h, __import__("ctypes").byref(ex), d_text.data_ptr(),
                                    d_offs.data_ptr(), n, d_w.data_ptr(), 0.0, P.MODE_EXACT,
                                    d_scores.data_ptr(), sh))

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        if world > 1 and dp is not None:
            # pars_dp_score_order: shard score + shard order, all-gather, each
            # rank places its own run, one uint32 all-reduce
            dp.score_order(ex, d_text.data_ptr(), d_offs.data_ptr(), N_PROMPTS, d_w.data_ptr(), 0.0,
                           P.MODE_EXACT, g_scores.data_ptr(), g_order.data_ptr(),
                           d_tie_all=g_tie.data_ptr(), stream=sh)
            if ev is not None:
                ev[1].record(stream)
                ev[2].record(stream)
            return
        score_shard()
        if ev is not None:
            ev[1].record(stream)
        check(L.pars_dev_priority_order(ctx.h, d_scores.data_ptr(), None, d_tie.data_ptr(), n,
                                        d_order.data_ptr(), sh))
        if world > 1:
            gather_into(g_pad, d_scores)
            gather_into(g_orders, d_order)
            if rank == 0:
                check(L.pars_dev_merge_orders(ctx.h, g_pad.data_ptr(), None, g_tie.data_ptr(),
                                              g_orders.data_ptr(), run_offs.ctypes.data, world,
                                              g_order.data_ptr(), sh))
        if ev is not None:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # full parity of this shard (untimed): every exact score bit-identical to
    # the oracle (the C restatement, threaded over the host cores) and the
    # shard's SJF order identical to the oracle's select_batch restatement
    from oracle.bind import Extractor as OEx
    from oracle.bind import Oracle
    o = Oracle()
    t_par = time.perf_counter()
    got = (g_scores[b:e] if world > 1 and dp is not None else d_scores[:n]).cpu().numpy()
    so = o.score_batch(OEx.make(), wl.text, wl.offsets[b:e + 1], w, 0.0, threads=host_threads())
    parity_ok = bool((got.view(np.uint64) == so.view(np.uint64)).all())
    if world > 1 and dp is not None:  # this rank's shard order, for the shard check
        check(L.pars_dev_priority_order(ctx.h, g_scores[b:].data_ptr(), None, d_tie.data_ptr(), n,
                                        d_order.data_ptr(), sh))
        torch.cuda.synchronize()
    got_order = d_order[:n].cpu().numpy().astype(np.int64)
    oorder = o.select_order(np.zeros(n), ["p%06d" % i for i in range(b, e)], so,
                            np.zeros(n, np.uint8), 0.0)
    order_ok = bool((got_order == oorder).all())
    t_par = time.perf_counter() - t_par
    outputs = None
    if world == 1:
        outputs = {"scores_sha256": hashlib.sha256(got.tobytes()).hexdigest()[:32],
                   "order_sha256": hashlib.sha256(got_order.tobytes()).hexdigest()[:32]}
    # the fast mode on the same prompts (fp32 products, tree reduction): its
    # kernel time and its order quality as Kendall tau_b against the exact
    # fp64 scores (GPU tau, metrics.cpp:42-64)
    fast = None
    if world == 1 and not args.no_configs:
        d_fast = torch.empty(n, dtype=torch.float64, device=dev)

        def score_fast():
            check(L.pars_dev_score_text(ctx.h, __import__("ctypes").byref(ex), d_text.data_ptr(),
                                        d_offs.data_ptr(), n, d_w.data_ptr(), 0.0, P.MODE_FAST,
                                        d_fast.data_ptr(), sh))
        fast_ms = timed_ms(torch, stream, 1, score_fast, args.steps)
        d_ex = torch.from_numpy(got).to(dev)
        tau_fe, _ = ctx.dev_kendall_tau(d_ex.data_ptr(), d_fast.data_ptr(), n, stream=sh)
        fs = d_fast.cpu().numpy()
        fast = {"kernel_ms": fast_ms, "prompts_per_s": n / (fast_ms / 1e3),
                "tau_b_vs_exact": tau_fe,
                "max_abs_diff_vs_exact": float(np.abs(fs - got).max()),
                "mode": "PARS_MODE_FAST_F32 (fp32 weights and products, tree reduction)"}
        del d_fast, d_ex
    global_order_ok = None
    if world > 1 and rank == 0:
        # the merged global order equals one sort of all N gathered scores
        full = torch.empty(N_PROMPTS, dtype=torch.int32, device=dev)
        gs = g_scores if dp is not None else g_pad
        L.pars_dev_priority_order(ctx.h, gs.data_ptr(), None, g_tie.data_ptr(), N_PROMPTS,
                                  full.data_ptr(), sh)
        torch.cuda.synchronize()
        global_order_ok = bool(torch.equal(full, g_order))

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
    if world > 1 and dp is not None:  # the fused dp step has no split: time the kernels alone
        feat_ms = timed_ms(torch, stream, 1, score_shard, args.steps)
        sort_ms = timed_ms(torch, stream, 1, lambda: check(L.pars_dev_priority_order(
            ctx.h, d_scores.data_ptr(), None, d_tie.data_ptr(), n, d_order.data_ptr(), sh)), args.steps)

    # roofline of the dominant kernel (fused featurize+score): algorithmic bytes
    alg_bytes = text_bytes + 8 * (n + 1) + 8 * n + 8 * DIM
    # ... and its integer-issue roofline: int ops counted on the
    # host from the text, sum over tokens of 4(l+1) + 12 max(0, l-2) + 8 per
    # emitted feature (one word + max(0, l-2) char trigrams per token), over
    # the measured integer issue peak (tools/micro/int_issue.cu)
    ntok, sum_len, sum_tri, _ = wl.token_stats(b, e)
    int_ops = 4 * (sum_len + ntok) + 12 * sum_tri + 8 * (ntok + sum_tri)
    spec_issue, meas_issue = issue_peaks()
    hbm, peak_kind = peaks()
    achieved = alg_bytes / (feat_ms / 1e3) / 1e9
    # traffic and pipe utilisation from the committed ncu capture of this
    # kernel (tools/profile_round.sh -> tools/ncu_to_json.py), scaled to this
    # launch's prompt count
    traffic, issue = None, None
    prof = ROOT / "profiles" / "featurize_ncu.json"
    if prof.exists():
        try:
            pj = json.loads(prof.read_text())
            traffic = pj["dram_bytes_per_prompt"] * n
            issue = {k: pj[k] for k in ("alu_pipe_pct_active", "fma_pipe_pct_active",
                                        "lsu_wavefronts_pct", "issue_active_pct",
                                        "dram_throughput_pct")}
            issue["source"] = "profiles/featurize_ncu.json (ncu --set full, %d prompts)" % pj["prompts"]
        except Exception:
            traffic, issue = None, None

    # e2e through the host-buffer C ABI (H2D text+offsets, D2H scores+order)
    ids_rank = np.arange(b, e, dtype=np.uint32)
    e2e_vals = []
    if n > 0 and not args.no_e2e:
        sub_offs = wl.offsets[b:e + 1]
        txt = wl.text  # pinned arena, offsets absolute
        # caller-owned page-locked result buffers, reused across steps like a
        # serving loop's: the scores and the order are DMA'd straight into them
        outs = (P.pinned_empty(e - b, np.float64), P.pinned_empty(e - b, np.int64))
        for k in range(max(1, args.e2e_steps) + 1):
            barrier(world)
            t0 = time.perf_counter()
            s, order = ctx.score_order(ex, txt, sub_offs, w, ids_rank, out=outs)
            t1 = time.perf_counter()
            if k > 0:
                e2e_vals.append(barrier_max(world, t1 - t0))
    e2e_s = float(np.median(e2e_vals)) if e2e_vals else float("nan")
    e2e_vals_ok = bool(e2e_vals)
    e2e_value = (N_PROMPTS if world > 1 else n) / e2e_s
    # the same step through the reference's public C++ API (Scorer::score_batch
    # over pageable std::string records + select_batch), linked with the
    # drop-in: a program written against proj/include only (tools/c4api_main.cpp)
    api_e2e = None
    if world == 1 and not args.no_e2e and n == N_PROMPTS:
        api_e2e = bench_reference_api(w, got, got_order)
    h2d = text_bytes + 8 * (n + 1) + 8 * DIM + 4 * n  # text, offsets, weights, tie ranks
    d2h = 8 * n + 4 * n  # scores, order

    # secondary: C5 all-pairs step (filtered pairs/s)
    configs = None
    if world == 1 and not args.no_configs:
        configs = bench_configs(P, ctx, args)
    pairs = None
    if not args.no_pairs:
        pairs = bench_pairs(P, ctx, torch, dev, stream, world, rank, args, dp)
    tau = None
    if not args.no_pairs:
        tau = bench_tau(P, ctx, torch, dev, stream, world, rank, args, dp)
    embed = None
    if world == 1 and not args.no_configs:
        embed = bench_embeddings(P, ctx, torch, dev, stream, args)
        embed["csr_gather"] = bench_csr_gather(P, ctx, torch, dev, stream, wl, w, d_scores, args)
        if configs is not None:
            configs["ingest_c4"] = bench_ingest(P, ctx, torch, dev, stream, wl, w, args)
            configs["c4_hard"] = bench_c4_hard(P, ctx, torch, dev, stream, w, args)

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            thr = host_threads()
            ref = CpuReferenceScoring(wl, w, args.cpu_sample, thr)
            ref.step()  # warm
            v = max(ref.step() for _ in range(3))  # best of 3
            cpu = {"value": v, "unit": "prompts/s", "cores": thr, "kind": "reference",
                   "cpu_model": cpu_model(),
                   "sample": f"first {ref.n} prompts of the same C4 workload: score_batch "
                             f"(OpenMP {thr} threads) + select_batch, best of 3"}
        line = {
            "metric": "prompts scored/s", "value": value, "unit": "prompts/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "C4: score + SJF-sort 1M synthetic prompts x 512 tokens "
                                   "(exact fp64 mode, bit-identical to the reference)",
                       "global_batch": N_PROMPTS, "seq_len": PAD_TOKENS,
                       "parallelism": f"shard{world}",
                       **({"global_order": "all-gather of shard scores + shard orders, merged on "
                                           "rank 0 (pars_dev_merge_orders), inside the step"}
                          if world > 1 else {}), "extractor": "hashed word{1}+char{3}, D=4096, L2",
                       "l2_flush": "inputs larger than L2 (%.2f GB text per rank)" % (text_bytes / 1e9)},
            "roofline": {"bound": "hbm", "kernel": "featurize_lane_kernel<exact, fused> (tokenise+hash+histogram+L2+dot)",
                         "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "peak_kind": peak_kind, "traffic": traffic, "issue_bound_evidence": issue,
                         "algorithmic_bytes_per_launch": alg_bytes, "kernel_ms": feat_ms,
                         "sort_ms": sort_ms,
                         "issue": {"bound": "int issue", "int_ops_per_launch": int_ops,
                                   "ops_model": "sum over tokens of 4(l+1) + 12 max(0,l-2) + 8 per "
                                                "emitted feature (SURVEY 8(d)), counted on the host "
                                                "from the text: %d tokens, %d token bytes, %d "
                                                "trigrams" % (ntok, sum_len, sum_tri),
                                   "achieved": int_ops / (feat_ms / 1e3) / 1e12,
                                   "peak": (meas_issue or spec_issue) / 1e12,
                                   "unit": "T int-ops/s",
                                   "frac": int_ops / (feat_ms / 1e3) / (meas_issue or spec_issue),
                                   "peak_kind": "measured: tools/micro/int_issue.cu fnv_step "
                                                "(LOP3+IMAD) mix, profiles/r2_int_issue.json"
                                                if meas_issue else "spec issue rate",
                                   "spec_peak": spec_issue / 1e12}},
            "sort": sort_roofline(n, sort_ms, hbm, got),
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "prompts/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "api": "pars_score_order (host buffers: score + SJF order in one call)"},
            "e2e_reference_api": api_e2e,
            "fast_mode": fast,
            "gpu_launches": int(launches),
            "clocks": clk,
            "parity": {"c4_scores_all": parity_ok, "c4_order_all": order_ok, "prompts_checked": n,
                       "check_s": t_par,
                       "oracle": "oracle/pars_oracle.c score_batch + select_batch restatement",
                       **({"global_order_equals_full_sort": global_order_ok} if world > 1 else {})},
            "outputs": outputs,
            "native_loaded": repo_native_loaded(),
            "workload_gen_s": t_gen,
        }
        # the bulky per-config detail goes on its own line first; the driver
        # reads the last line, which stays compact
        print(json.dumps({"detail": True, "pairs": pairs, "kendall_tau": tau,
                          "embeddings": embed, "configs": configs}))
        if pairs is not None:
            print(json.dumps({"metric": "filtered pairs/s", "value": pairs["value"],
                              "unit": "pairs/s", "n_gpus": world,
                              "ms_per_step": pairs["ms_per_step"], "config": "C5"}))
        print(json.dumps(line))
    if dp is not None:
        dp.close()
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def make_dp(P, ctx, world, rank):
    """The C ABI's NCCL data-parallel layer (pars_dp_*): one communicator per
    rank, its unique id broadcast from rank 0. None in the gloo test mode
    (several ranks on one GPU, which NCCL refuses)."""
    if os.environ.get("PARS_DIST_BACKEND", "nccl") != "nccl":
        return None
    uid = P.nccl_unique_id() if rank == 0 else bytes(128)
    if world > 1:
        import torch.distributed as dist
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    return P.DataParallel(ctx, uid, world, rank)


def timed_ms(torch, stream, world, fn, k):
    """Mean device time of fn() over k calls on `stream` (CUDA events),
    max over ranks."""
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    barrier(world)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(k):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return barrier_max(world, a.elapsed_time(b)) / k


def sort_roofline(n, sort_ms, hbm, scores=None):
    """The priority sort's HBM roofline: the one-pass I/O floor (read score +
    tie rank, write the order) and, beside it, the passes it actually runs.
    LSD passes run per score byte position where the keys differ (C4's burst
    tie ranks are already in input order, so the 4 tie-rank positions are
    skipped), each moving the 8 B key + 4 B index in and out (24 B per key);
    when two or more of the low four byte positions are active, the passes
    over the top four run first and radix_fixup orders runs of equal top
    words (16 B per key: key + index read, order written) — held if no run
    is longer than 32 keys, else the full LSD passes run as well."""
    floor = n * (8 + 4 + 4)
    out = {"kernel": "radix sort (pars_dev_priority_order)", "ms": sort_ms, "bound": "hbm",
           "floor_bytes": floor, "bytes_model": "one-pass I/O floor: 8 B score + 4 B tie rank "
           "read, 4 B order written per key",
           "achieved": floor / (sort_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
           "frac": floor / (sort_ms / 1e3) / 1e9 / hbm}
    if scores is not None and len(scores):
        b = np.ascontiguousarray(scores, np.float64).view(np.uint64).copy()
        b[(b << np.uint64(1)) == 0] = 0  # -0.0 == +0.0
        neg = (b >> np.uint64(63)) == 1
        key = np.where(neg, ~b, b | np.uint64(1 << 63))
        act = [int(np.unique((key >> np.uint64(8 * p)) & np.uint64(0xff)).size > 1) for p in range(8)]
        lo_act, hi_act = sum(act[:4]), sum(act[4:])
        spec = hi_act > 0 and lo_act >= 2
        longest = int(np.unique(key >> np.uint64(32), return_counts=True)[1].max()) if spec else 0
        held = spec and longest <= 32
        passes = hi_act if held else lo_act + hi_act + (hi_act if spec else 0)
        moved = passes * n * 24 + (n * 16 if spec else 0)
        out.update({"passes": passes, "high_word_speculation": spec, "fixup_held": held,
                    "longest_top_word_run": longest, "pass_bytes": moved,
                    "pass_model": "24 B per key per radix pass (8 B key + 4 B index, read and "
                                  "written) + 16 B per key for the fixup when speculating",
                    "pass_achieved": moved / (sort_ms / 1e3) / 1e9,
                    "pass_frac": moved / (sort_ms / 1e3) / 1e9 / hbm})
    return out


def issue_peaks():
    """Lane-op issue peaks: the spec rate (one warp-instruction per cycle per
    SM sub-partition at the max SM clock) and the measured integer mix of the
    featurize hash (tools/micro/int_issue.cu -> profiles/r2_int_issue.json)."""
    mp = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    clk = float(mp.get("sm_max_mhz", 1965.0)) * 1e6
    spec = 148 * 4 * 32 * clk
    meas = None
    p = ROOT / "profiles" / "r2_int_issue.json"
    if p.exists():
        try:
            meas = float(json.loads(p.read_text())["kinds"]["fnv_step (LOP3+IMAD)"]["lane_ops_per_s"])
        except Exception:
            meas = None
    return spec, meas


def bench_pairs(P, ctx, torch, dev, stream, world, rank, args, dp=None):
    """C5: one full-batch data-parallel training step over 65,536 prompts
    through pars_dp_train_step: score this rank's prompt shard (exact CSR
    dot), all-gather the scores, this rank's cost-balanced slice of the
    all-pairs tiles (Eq. 1 mask + hinge + integer coefficients), all-reduce
    the coefficients and counts, X^T c on the row shard, all-reduce the
    gradient, w -= (lr / kept) * grad (a kernel). Metric: kept pairs per
    second of step time (max over ranks)."""
    wl = P.Workload.synthesize(C5_N, C5_SEED)
    ex = P.Extractor.make()
    feats = ctx.extract(ex, wl.text, wl.offsets)  # once, like train()'s extract_all
    n = C5_N
    w0 = np.random.default_rng(99).normal(size=DIM) * 0.05
    d_w = torch.from_numpy(w0).to(dev)
    sh = stream.cuda_stream
    plan = ctx.pair_plan(wl.output_len, DELTA)  # per dataset: lengths are fixed
    kept = plan.kept
    lr = 0.1
    d_s = torch.empty(n, dtype=torch.float64, device=dev)
    d_c = torch.zeros(n, dtype=torch.int32, device=dev)
    d_cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    d_loss = torch.zeros(1, dtype=torch.float64, device=dev)
    if dp is not None:
        def step():
            dp.train_step(feats, plan, d_w.data_ptr(), MARGIN, lr, d_c.data_ptr(), d_s.data_ptr(),
                          d_cnt.data_ptr(), d_loss.data_ptr(), stream=sh)
    else:  # gloo test mode: the torch.distributed restatement (distributed.py)
        from paper_2510_03243_b200 import distributed as D
        lens = wl.output_len.astype(np.int32)
        d_L = torch.from_numpy(lens).to(dev)
        per = (n + world - 1) // world
        scores_pad = torch.zeros(per * world, dtype=torch.float64, device=dev)

        def step():
            cnt, part = D.train_step_gpu(ctx, feats, d_w, scores_pad, d_L, n, DELTA, MARGIN,
                                         int(lens.max()), lr / kept, stream=sh, plan=plan)
            d_cnt.copy_(cnt)
            d_s.copy_(scores_pad[:n])

    # parity of the first step (untimed, from w0) against the oracle: scores
    # and integer coefficients bit-exact, counts exact, the loss and the
    # updated weights within the stated tolerances (fp64 sums in another order)
    from oracle.bind import Extractor as OEx
    from oracle.bind import Oracle
    o = Oracle()
    step()
    torch.cuda.synchronize()
    so = o.score_batch(OEx.make(), wl.text, wl.offsets, w0, 0.0, threads=host_threads())
    oc, okept, oact, oloss = o.allpairs(so, wl.output_len, DELTA, MARGIN, threads=host_threads())
    par = {"c5_scores": bool((d_s.cpu().numpy().view(np.uint64) == so.view(np.uint64)).all()),
           "c5_kept": int(d_cnt[0]) == okept == 1920977782, "c5_active": int(d_cnt[1]) == oact}
    if dp is not None:
        rp, idx, val = feats.download()
        g = o.xt_c(rp, idx, val, oc, DIM)
        rows = np.repeat(np.arange(n), np.diff(rp))
        mag = np.zeros(DIM)
        np.add.at(mag, idx, np.abs(val * oc[rows]))
        w1 = w0 - (lr / okept) * g
        dw = np.abs(d_w.cpu().numpy() - w1)
        scale = (lr / okept) * mag
        grad_rel = float(np.max(np.where(scale > 0, dw / np.where(scale > 0, scale, 1), 0.0)))
        loss_rel = abs(float(d_loss[0]) - oloss) / abs(oloss)
        par.update({"c5_coeff": bool((d_c.cpu().numpy() == oc).all()),
                    "c5_loss_rel": loss_rel, "c5_grad_rel": grad_rel,
                    "tolerance": "loss <= 1e-12 relative; weights |w - w_oracle| <= 1e-12 * "
                                 "(lr/kept) * sum_i |c_i x_i[d]| per component (X^T c summed "
                                 "in another order)",
                    "c5_ok": bool(loss_rel <= 1e-12 and grad_rel <= 1e-12)})
        del rp, idx, val, rows
    first_ok = all(v for k, v in par.items() if isinstance(v, bool))
    d_w.copy_(torch.from_numpy(w0).to(dev))
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    # the whole step (kernels and NCCL collectives) as one CUDA graph replayed
    # per step: the host launches nothing per kernel. Falls back to eager
    # launches if capture is refused.
    graph = None
    if dp is not None:
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step()
            graph = g
        except Exception as exc:  # noqa: BLE001
            print("bench_pairs: CUDA graph capture failed (%s); timing eager steps" % exc,
                  file=sys.stderr)
            graph = None
            torch.cuda.synchronize()
    run = graph.replay if graph is not None else step
    k = max(3, args.steps)
    ms = timed_ms(torch, stream, world, run, k)
    graph_ok = None
    if graph is not None:
        # replaying the graph trains exactly like launching the steps
        d_w.copy_(torch.from_numpy(w0).to(dev))
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        w_graph = d_w.clone()
        d_w.copy_(torch.from_numpy(w0).to(dev))
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        graph_ok = bool(torch.equal(w_graph.view(torch.int64), d_w.view(torch.int64)))
    active = int(d_cnt[1])
    # the dominant kernel alone, over every tile (prep + allpairs + scatter),
    # and X^T c over every row, each timed with events on the launch stream
    tiles = int(P.lib().pars_allpairs_tiles(n))
    part = torch.zeros(tiles, dtype=torch.float64, device=dev)
    ms_pairs = timed_ms(torch, stream, world, lambda: plan.run(
        d_s.data_ptr(), MARGIN, 0, tiles, d_c.data_ptr(), d_cnt.data_ptr(), part.data_ptr(), sh), k)
    d_g = torch.zeros(DIM, dtype=torch.float64, device=dev)
    L = P.lib()
    ms_xtc = timed_ms(torch, stream, world, lambda: L.pars_dev_xt_c(
        ctx.h, __import__("ctypes").c_void_p(feats.h), d_c.data_ptr(), 0, n, d_g.data_ptr(), sh), k)
    nnz = feats.nnz
    spec, meas = issue_peaks()
    all_pairs = n * (n - 1) // 2
    ach = all_pairs * 11 / (ms_pairs / 1e3)
    hbm, peak_kind = peaks()
    xtc_bytes = nnz * 12 + (DIM + 1) * 8 + n * 4 + DIM * 8
    feats.free()
    return {"metric": "filtered pairs/s", "value": kept / (ms / 1e3), "unit": "pairs/s",
            "ms_per_step": ms, "kept": kept, "kept_expected": 1920977782,
            "active_last_step": active, "first_step_matches_oracle": first_ok, "parity": par,
            "plan_sorted": plan.sorted, "cuda_graph": graph is not None,
            "cuda_graph_matches_eager": graph_ok,
            "api": "pars_dp_train_step (NCCL world %d)" % world if dp is not None else
                   "distributed.train_step_gpu (gloo test mode)",
            "workload": "C5: full-batch DP training step over all 2,147,450,880 unordered pairs "
                        "of 65,536 prompts (seed 25): CSR scoring of the rank's shard + score "
                        "all-gather, Eq.1 mask delta=0.2 + hinge + integer coefficients on the "
                        "rank's tiles + all-reduce, X^T c + gradient all-reduce, SGD update",
            "bound": "issue (int/fp64 ALU); inputs 0.5 MB are L2-resident",
            "roofline": {"bound": "issue", "kernel": "allpairs_sorted_kernel (+ prep, scatter), "
                         "all tiles on one GPU", "kernel_ms": ms_pairs,
                         "achieved": ach / 1e12, "peak": spec / 1e12, "unit": "T lane-ops/s",
                         "frac": ach / spec,
                         "algorithmic": "11 lane-ops per unordered pair (SURVEY 8(d): sub, abs, "
                                        "max, dmin lookup, compare, label, sign, add-margin, max, "
                                        "2 accumulates) x all 2,147,450,880 pairs; the sorted "
                                        "plan executes far fewer: empty tiles are skipped, "
                                        "tiles the Eq. 1 mask keeps whole (all but the diagonal "
                                        "and mask-boundary tiles) are counted by two 8-step "
                                        "binary searches per row/column over per-tile sorted "
                                        "scores and thresholds, the rest by one compare per "
                                        "pair; so frac exceeds 1 (pair-equivalent rate)",
                         "peak_kind": "spec: 148 SMs x 4 SMSPs x 32 lanes x max SM clock",
                         "measured_int_mix_peak": meas / 1e12 if meas else None,
                         "pairs_per_s_kernel": all_pairs / (ms_pairs / 1e3)},
            "xtc": {"kernel": "xtc_csc_kernel + xtc_task_reduce (grad = X^T c, all 65,536 rows)",
                    "ms": ms_xtc, "bound": "hbm", "algorithmic_bytes": xtc_bytes,
                    "bytes_model": "nnz x (4 B row + 8 B value) + column pointers + c + grad",
                    "achieved": xtc_bytes / (ms_xtc / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                    "frac": xtc_bytes / (ms_xtc / 1e3) / 1e9 / hbm, "peak_kind": peak_kind}}


def bench_tau(P, ctx, torch, dev, stream, world, rank, args, dp=None):
    """Kendall tau-b counts (metrics.cpp:42-64) at compare_policies scale: the
    PARS scores vs output lengths of 100,000 requests (C3-sized trace). The
    default path counts by sorting (tau_sorted.cu, O(n log n), exact; every
    rank computes the whole trace, no collective); the all-pairs tile path
    (4,999,950,000 pairs split over ranks + one exact all-reduce) is timed
    beside it. value = all-pairs-equivalent pairs per second."""
    from paper_2510_03243_b200 import distributed as D
    n = 100_000
    wl = P.Workload.synthesize(n, 23)
    w = np.random.default_rng(5).normal(size=DIM) * 0.05
    s = ctx.score_text(P.Extractor.make(), wl.text, wl.offsets, w)
    y = wl.output_len.astype(np.float64)
    dx, dy = torch.from_numpy(s).to(dev), torch.from_numpy(y).to(dev)
    sh = stream.cuda_stream
    k = max(3, args.steps)

    def timed(fn):
        for _ in range(2):
            r = fn()
        torch.cuda.synchronize()
        barrier(world)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(k):
            r = fn()
        b.record(stream)
        torch.cuda.synchronize()
        return barrier_max(world, a.elapsed_time(b)) / k, r

    ms, (tau, c) = timed(lambda: ctx.dev_kendall_tau(dx.data_ptr(), dy.data_ptr(), n, stream=sh))
    if dp is not None:  # pars_dp_kendall_tau: tiles split over ranks, one u64 all-reduce
        ms_pairs, (tau_p, c_p) = timed(lambda: dp.kendall_tau(dx.data_ptr(), dy.data_ptr(), n, stream=sh))
    else:
        ms_pairs, (tau_p, c_p) = timed(lambda: D.kendall_tau_gpu(ctx, dx, dy, n, stream=sh))
    pairs = n * (n - 1) // 2
    out = {"metric": "pairs/s", "value": pairs / (ms / 1e3), "ms_per_call": ms, "tau_b": tau,
           "algorithm": "sorted counts (two radix sorts + merge inversion count, replayed as one CUDA graph), exact",
           "roofline": {"bound": "latency", "floor_bytes": 16 * n + 32,
                        "bytes_model": "one-pass I/O floor: x and y (8 B each) read once, 4 counts written",
                        "achieved": (16 * n + 32) / (ms / 1e3) / 1e9, "peak": peaks()[0], "unit": "GB/s",
                        "frac": (16 * n + 32) / (ms / 1e3) / 1e9 / peaks()[0],
                        "note": "the two stable radix sorts (sort roofline) and log2(n) merge levels are "
                                "dependent launches on 0.8 MB of L2-resident data"},
           "pairs_path_ms": ms_pairs, "pairs_path_pairs_per_s": pairs / (ms_pairs / 1e3),
           "paths_agree": bool((c == c_p).all()) and tau == tau_p,
           "workload": "kendall_tau_b(scores, output_len) over 100,000 requests "
                       "(4,999,950,000 pairs), exact integer counts"}
    if world == 1 and not args.no_cpu:
        from oracle.bind import Oracle
        m = 30_000
        t0 = time.perf_counter()
        otau, oc = Oracle().kendall(s[:m], y[:m], threads=host_threads())
        dt = time.perf_counter() - t0
        gt, gc = ctx.dev_kendall_tau(dx[:m].contiguous().data_ptr(), dy[:m].contiguous().data_ptr(),
                                     m, stream=sh)
        out.update({"cpu_pairs_per_s": (m * (m - 1) // 2) / dt, "cpu_threads": host_threads(),
                    "cpu_sample": "first %d requests (port of metrics.cpp, OpenMP)" % m,
                    "sample_counts_match": bool((gc == oc).all()) and gt == otau})
    return out


def bench_c4_hard(P, ctx, torch, dev, stream, w, args):
    """SURVEY 8(d)'s hard C4 variant: prompts padded to 512 tokens with random
    6-letter words (~3.4 KB, ~1,520 touched buckets per prompt). A 200,000-
    prompt sample (0.69 GB of text, device-resident), exact and fast modes,
    parity of the first 2,000 exact scores against the oracle, and the
    reference's score_batch on 2,000 prompts on all host threads."""
    import ctypes as C
    from oracle.bind import Extractor as OEx
    from oracle.bind import Oracle
    n = 200000
    hw = P.Workload.synthesize(n, SEED, pad_tokens=PAD_TOKENS, pad_seed=PAD_SEED, pad_words="random6")
    d_text = torch.from_numpy(hw.text[: int(hw.offsets[-1])]).to(dev)
    d_offs = torch.from_numpy(hw.offsets).to(dev)
    d_w = torch.from_numpy(w).to(dev)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    ex = P.Extractor.make()
    L = P.lib()
    sh = stream.cuda_stream
    res = {"workload": "C4 hard variant: %d prompts padded to 512 tokens with random 6-letter words" % n,
           "bytes_per_prompt": float(hw.offsets[-1]) / n}
    for name, mode in (("exact", P.MODE_EXACT), ("fast", P.MODE_FAST)):
        def step():
            rc = L.pars_dev_score_text(ctx.h, C.byref(ex), d_text.data_ptr(), d_offs.data_ptr(), n,
                                       d_w.data_ptr(), 0.0, mode, out.data_ptr(), sh)
            if rc != 0:
                raise P.ParsError(rc, L.pars_last_error().decode("utf-8", "replace"))
        ms = timed_ms(torch, stream, 1, step, max(args.steps, 3))
        res[name + "_ms_per_1M"] = ms * 1e6 / n
        res[name + "_prompts_per_s"] = n / (ms / 1e3)
        if name == "exact":
            got = out[:2000].cpu().numpy()
            want = Oracle().score_batch(OEx.make(), hw.text, hw.offsets[:2001], w, 0.0,
                                        threads=host_threads())
            res["exact_bitexact_sample"] = bool((got.view(np.uint64) == want.view(np.uint64)).all())
            res["sample"] = 2000
    if not args.no_cpu:
        t0 = time.perf_counter()
        Oracle().score_batch(OEx.make(), hw.text, hw.offsets[:2001], w, 0.0, threads=host_threads())
        res["cpu_prompts_per_s"] = 2000 / (time.perf_counter() - t0)
        res["cpu_threads"] = host_threads()
        res["cpu_kind"] = "port (oracle/pars_oracle.c score_batch, OpenMP)"
    del d_text, d_offs, out
    return res


def bench_csr_gather(P, ctx, torch, dev, stream, wl, w, d_scores, args):
    """Repeated scoring over precomputed features (SURVEY 8(d) 'sparse
    gather-dot over CSR'): extract_all of the 1 M C4 prompts once (untimed),
    then pars_dev_features_score over all rows — each row's exact dot
    (features.hpp:31-35) from the compact rows (idx << 16 | count16, 4 B per
    entry, v = count * inv recomputed with the same __dmul_rn). HBM-bound:
    the bytes it moves are the compact entries + per-row metadata + scores."""
    import ctypes as C
    n = len(wl.offsets) - 1
    f = ctx.extract(P.Extractor.make(), wl.text, wl.offsets)
    rp = f.download()[0]
    nnz = int(rp[-1])
    d_w = torch.from_numpy(w).to(dev)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    L = P.lib()
    sh = stream.cuda_stream

    def step():
        rc = L.pars_dev_features_score(ctx.h, C.c_void_p(f.h), 0, n, d_w.data_ptr(), 0.0, out.data_ptr(), sh)
        if rc != 0:
            raise P.ParsError(rc, L.pars_last_error().decode("utf-8", "replace"))

    ms = timed_ms(torch, stream, 1, step, max(args.steps, 5))
    same = bool(torch.equal(out.view(torch.int64), d_scores[:n].view(torch.int64)))
    f.free()
    hbm, kind = peaks()
    moved = nnz * 4 + n * (8 + 4 + 8 + 8)
    model = nnz * 12 + n * 16
    return {"metric": "prompts scored/s", "value": n / (ms / 1e3), "unit": "prompts/s", "ms_per_step": ms,
            "nnz": nnz, "workload": "pars_dev_features_score over the 1 M C4 prompts' precomputed features",
            "bit_identical_to_text_path": same,
            "roofline": {"bound": "hbm", "algorithmic_bytes": moved,
                         "bytes_model": "compact entries 4 B/nnz + row pointer 8 B + entry offset 4 B + "
                                        "inverse norm 8 B + score 8 B per row",
                         "achieved": moved / (ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": moved / (ms / 1e3) / 1e9 / hbm, "peak_kind": kind,
                         "survey_model_bytes": model,
                         "survey_model_note": "SURVEY 8(d) counts a 4 B index + 8 B value per nnz; the "
                                              "compact format moves 4 B per nnz"}}


def bench_embeddings(P, ctx, torch, dev, stream, args):
    """PrecomputedEmbedding scoring (features.cpp:67-76 + L2 + dot), exact
    fp64 mode, device-resident rows: 65,536 prompts x 4,096 dims (2.1 GB,
    larger than L2). HBM-bound: algorithmic bytes = the rows once + weights +
    scores; the exact path streams the rows twice (sum of squares first, then
    the dot, both in index order), so its ceiling is 0.5 of the roofline."""
    import ctypes as C
    n, dim = 65536, DIM
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    X = torch.randn(n, dim, dtype=torch.float64, device=dev, generator=g)
    w = torch.randn(dim, dtype=torch.float64, device=dev, generator=g)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    ex = P.Extractor.make(dim=dim, kind="embedding", norm="l2")
    L = P.lib()
    sh = stream.cuda_stream

    def step():
        rc = L.pars_dev_score_embeddings(ctx.h, C.byref(ex), X.data_ptr(), n, w.data_ptr(), 0.0,
                                         P.MODE_EXACT, out.data_ptr(), sh)
        if rc != 0:
            raise P.ParsError(rc, L.pars_last_error().decode("utf-8", "replace"))

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    # parity spot check against the oracle on the first rows (untimed)
    from oracle.bind import Extractor as OEx
    from oracle.bind import Oracle
    chk = 256
    want = Oracle().score_dense(OEx.make(dim=dim, kind="embedding", norm="l2"),
                                X[:chk].cpu().numpy(), w.cpu().numpy(), 0.0)
    ok = bool((out[:chk].cpu().numpy().view(np.uint64) == want.view(np.uint64)).all())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = max(3, args.steps)
    a.record(stream)
    for _ in range(k):
        step()
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / k
    alg = n * dim * 8 + dim * 8 + n * 8
    hbm, _ = peaks()
    ach = alg / (ms / 1e3) / 1e9
    exact = out.clone()
    # fast mode (fp32 products, tree reductions, one pass over the rows)
    w32_rel = None

    def step_fast():
        rc = L.pars_dev_score_embeddings(ctx.h, C.byref(ex), X.data_ptr(), n, w.data_ptr(), 0.0,
                                         P.MODE_FAST, out.data_ptr(), sh)
        if rc != 0:
            raise P.ParsError(rc, L.pars_last_error().decode("utf-8", "replace"))
    ms_fast = timed_ms(torch, stream, 1, step_fast, k)
    # tolerance: |fast - exact| <= 1e-5 * sum_i |w_i v_i|
    Xn = X / X.norm(dim=1, keepdim=True)
    mag = (Xn.abs() * w.abs()).sum(dim=1)
    w32_rel = float(((out - exact).abs() / mag).max())
    tau_fe, _ = ctx.dev_kendall_tau(exact.data_ptr(), out.data_ptr(), n, stream=sh)
    del Xn
    ach_fast = alg / (ms_fast / 1e3) / 1e9
    return {"metric": "prompts scored/s", "value": n / (ms / 1e3), "unit": "prompts/s",
            "ms_per_step": ms, "parity_bitexact_sample": ok, "sample": chk,
            "workload": "PrecomputedEmbedding: 65,536 prompts x 4,096 fp64 dims, L2 norm, exact",
            "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                         "frac": ach / hbm, "algorithmic_bytes_per_launch": alg,
                         "note": "exact mode reads the rows twice (norm chain, then dot chain): "
                                 "its ceiling is 0.5 of this roofline"},
            "fast": {"ms_per_step": ms_fast, "value": n / (ms_fast / 1e3),
                     "roofline": {"bound": "hbm", "achieved": ach_fast, "peak": hbm, "unit": "GB/s",
                                  "frac": ach_fast / hbm,
                                  "note": "peak is the measured copy (read+write) bandwidth; this kernel "
                                          "only reads, and a read-only stream runs above it (frac against "
                                          "the 8,000 GB/s nominal HBM3e figure: %.2f)" % (ach_fast / 8000.0)},
                     "max_err_over_sum_abs_wv": w32_rel, "tolerance": 1e-5,
                     "tau_b_vs_exact": tau_fe}}


def bench_ingest(P, ctx, torch, dev, stream, wl, w, args):
    """From JSONL bytes to the SJF order: the C4 workload written as a
    pars.dataset file (1M records, ~2.2 GB), loaded by the GPU loader
    (pars_load_dataset_bytes: H2D of the bytes, line split, JSON validation,
    decoded prompt arena), scored and ordered on the device. Beside it the
    reference's load_dataset + score_batch + select_batch on the first 100k
    records of the same file (bounded sample)."""
    import ctypes as C
    import tempfile
    n = len(wl)
    head = b'{"embedding_dim":0,"format":"pars.dataset","version":1}\n'
    parts = [head]
    for i in range(n):
        parts.append(b'{"id":"p%07d","output_len":%d,"prompt":"' % (i, int(wl.output_len[i])))
        parts.append(wl.text[wl.offsets[i]:wl.offsets[i + 1]].tobytes())
        parts.append(b'"}\n')
    blob = b"".join(parts)
    nbytes = len(blob)
    hb = C.c_void_p()
    if P.lib().pars_host_alloc(nbytes, C.byref(hb)) != 0:
        raise MemoryError("pinned host allocation failed")
    host = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(hb.value))
    host[:] = np.frombuffer(blob, np.uint8)
    del blob, parts
    L = P.lib()
    ex = P.Extractor.make()
    d_w = torch.from_numpy(w).to(dev)
    d_s = torch.empty(n, dtype=torch.float64, device=dev)
    d_tie = torch.arange(n, dtype=torch.int32, device=dev)
    d_o = torch.empty(n, dtype=torch.int32, device=dev)
    sh = stream.cuda_stream

    def step():
        h = C.c_void_p()
        rc = L.pars_load_dataset_bytes(ctx.h, b"c4.jsonl", C.c_char_p(hb.value), nbytes, -1, C.byref(h))
        if rc != 0:
            raise P.ParsError(rc, L.pars_last_error().decode("utf-8", "replace"))
        g = P._lib.GpuDataset(h.value)
        L.pars_dev_score_text(ctx.h, C.byref(ex), g.dev_text, g.dev_offsets, len(g), d_w.data_ptr(),
                              0.0, P.MODE_EXACT, d_s.data_ptr(), sh)
        L.pars_dev_priority_order(ctx.h, d_s.data_ptr(), None, d_tie.data_ptr(), len(g),
                                  d_o.data_ptr(), sh)
        torch.cuda.synchronize()
        g.free()

    step()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    t = float(np.median(ts))
    out = {"workload": "C4 as a pars.dataset JSONL (%d records, %.2f GB): GPU load "
                       "(pars_load_dataset_bytes, bytes in pinned host memory) + score + SJF order"
                       % (n, nbytes / 1e9),
           "gpu_s": t, "gpu_records_per_s": n / t}
    if not args.no_cpu:
        from oracle.bind import Extractor as OEx
        from oracle.bind import Ref
        R = Ref()
        R.set_threads(host_threads())
        path = tempfile.mktemp(suffix=".jsonl")
        sample = 100_000
        with open(path, "wb") as f:
            f.write(host.tobytes())
        t0 = time.perf_counter()
        ds = R.load_dataset(path, sample)
        t_load = time.perf_counter() - t0
        rs = R.score_batch(OEx.make(), ds, w)
        R.select_batch(np.zeros(len(ds)), ["p%07d" % i for i in range(len(ds))], rs,
                       np.zeros(len(ds), np.uint8), 0.0, len(ds))
        t_all = time.perf_counter() - t0
        os.unlink(path)
        out.update({"cpu_records_per_s": sample / t_all, "cpu_load_s": t_load, "cpu_total_s": t_all,
                    "cpu_sample": "first %d records: load_dataset (1 thread, as the reference) + "
                                  "score_batch (OpenMP %d threads) + select_batch"
                                  % (sample, host_threads())})
    P.lib().pars_host_free(hb)
    return out


def bench_reference_api(w, scores, order):
    """C4 end to end through the reference API: oracle/_ref/c4api_b200 (the
    program tools/c4api_main.cpp — reference headers only — built against the
    drop-in libpars_b200.so; the reference's own generator makes the records).
    Its step is the reference arm's step; its outputs must equal ours."""
    import tempfile
    exe = ROOT / "oracle" / "_ref" / "c4api_b200"
    if not exe.exists():
        return {"unavailable": "oracle/_ref/c4api_b200 not built"}
    with tempfile.TemporaryDirectory() as td:
        wf = Path(td) / "w.bin"
        np.ascontiguousarray(w, np.float64).tofile(wf)
        pre = Path(td) / "out"
        r = subprocess.run([str(exe), str(N_PROMPTS), str(wf), "3", str(pre)], capture_output=True,
                           text=True, timeout=900)
        if r.returncode != 0:
            return {"error": (r.stderr or r.stdout)[-400:]}
        j = json.loads(r.stdout.strip().splitlines()[-1])
        s2 = np.fromfile(str(pre) + ".scores", np.float64)
        o2 = np.fromfile(str(pre) + ".order", np.int64)
    j["scores_equal_c_abi"] = bool(len(s2) == len(scores) and
                                   (s2.view(np.uint64) == scores.view(np.uint64)).all())
    j["order_equal_c_abi"] = bool(len(o2) == len(order) and (o2 == order).all())
    j["api"] = ("LinearScorer::score_batch(Dataset) + select_batch (proj/include/pars) "
                "through libpars_b200.so; records are pageable std::string")
    return j


def fnv64(a: np.ndarray) -> str:
    h = 0xCBF29CE484222325
    for b in a.astype("<u8" if a.dtype != np.float64 else "<f8").tobytes():
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def bench_configs(P, ctx, args):
    """BASELINE configs C1 and C2 (1 GPU, host-buffer API, latency-bound) and
    the CPU side of C5, each next to the reference CPU path on this host and
    with its golden parity anchor."""
    out = {}
    thr = host_threads()
    ex = P.Extractor.make()
    have_ref = not args.no_cpu
    if have_ref:
        from oracle.bind import Extractor as OEx
        from oracle.bind import Oracle, Ref
        R = Ref()
        R.set_threads(thr)
    # ---- C1: README model, score 1,024 prompts (<=128 tokens) + SJF order
    full = P.Workload.synthesize(4000, 21)
    # split_dataset(0.2, 21) of the reference: train part, restated through the
    # reference library when available (the model itself is trained on the GPU)
    if have_ref:
        rfull = R.synthesize(4000, 21)
        tr, _ = R.split(rfull, 0.2, 21)
        t0 = time.perf_counter()
        w, _, lt = ctx.train_pairwise(ex, tr.text, tr.offs, tr.output_len, seed=21)
        t_train = time.perf_counter() - t0
        g = P.Workload.synthesize(2048, 22)
        sel = np.nonzero(g.prompt_len <= 128)[0][:1024]
        arena, offs = P.pack_texts([g.prompt(i) for i in sel])
        ids = ["p%06d" % i for i in sel]
        tie = P.tie_ranks(np.zeros(len(sel)), ids)
        lat = []
        for k in range(13):
            t0 = time.perf_counter()
            sc = ctx.score_text(ex, arena, offs, w)
            order = ctx.priority_order(sc, tie)
            lat.append(time.perf_counter() - t0)
        gpu_ms = 1e3 * float(np.median(lat[3:]))
        # the same through the fused call (enqueue + select_batch, one sync)
        latf = []
        for k in range(13):
            t0 = time.perf_counter()
            scf, orderf = ctx.score_order(ex, arena, offs, w, tie)
            latf.append(time.perf_counter() - t0)
        fused_ms = 1e3 * float(np.median(latf[3:]))
        fused_same = bool((scf.view(np.uint64) == sc.view(np.uint64)).all() and (orderf == order).all())
        c1 = R.subset(g_ref := R.synthesize(2048, 22), sel)
        R.score_batch(OEx.make(), c1, w)
        cl = []
        for _ in range(5):
            t0 = time.perf_counter()
            rs = R.score_batch(OEx.make(), c1, w)
            R.select_batch(np.zeros(len(sel)), ids, rs, np.zeros(len(sel), np.uint8), 0.0, len(sel))
            cl.append(time.perf_counter() - t0)
        out["c1"] = {"workload": "score 1,024 prompts (<=128 tokens) + SJF order, README model",
                     "gpu_ms": fused_ms, "gpu_prompts_per_s": len(sel) / (fused_ms / 1e3),
                     "api": "pars_score_order (host buffers, one call)",
                     "gpu_ms_two_calls": gpu_ms, "fused_equals_two_calls": fused_same,
                     "cpu_ms": 1e3 * float(np.median(cl)), "cpu_threads": thr,
                     "scores_fnv": fnv64(sc), "order_fnv": fnv64(order.astype(np.uint64)),
                     "parity_bitexact": fnv64(sc) == "5548c3b3d81d615d"
                     and fnv64(order.astype(np.uint64)) == "e6e78f54425df769",
                     "readme_model_train_ms": 1e3 * t_train,
                     "readme_weights_fnv": fnv64(w),
                     "readme_weights_bitexact": fnv64(w) == "db7217cbd5a86b9b"}
    # ---- C2: one training epoch on 8,192 samples
    d2 = P.Workload.synthesize(8192, 21)
    ts = []
    for k in range(4):
        t0 = time.perf_counter()
        w2, _, lt2 = ctx.train_pairwise(ex, d2.text, d2.offsets, d2.output_len, seed=21, epochs=1)
        ts.append(time.perf_counter() - t0)
    gpu_epoch_ms = 1e3 * float(np.median(ts[1:]))
    c2 = {"workload": "one margin-ranking epoch, 8,192 samples, 100k pairs, delta 0.2 "
                      "(extract_all + build_pairs + 782 SGD steps)",
          "gpu_epoch_ms": gpu_epoch_ms, "gpu_pairs_per_s": 100000 / (gpu_epoch_ms / 1e3),
          "loss0": float(lt2[0]).hex(), "weights_fnv": fnv64(w2),
          "parity_bitexact": fnv64(w2) == "f97c96a353829ee2"
          and float(lt2[0]).hex() == "0x1.1b1e92d7700cap-1"}
    # the SGD epoch alone against its latency floor: every step's score
    # chains run in parallel, so a step is at least its longest chain of
    # dependent __dadd_rn (8 cycles each, tools/micro/fp64_latency.cu)
    f2 = ctx.extract(ex, d2.text, d2.offsets)
    a2, b2, y2, _ = P.build_pairs(d2.output_len, 0.2, 100000, 12345)
    nnz2 = np.diff(f2.download()[0])
    bt = 128
    longest = [int(max(nnz2[a2[q:q + bt]].max(), nnz2[b2[q:q + bt]].max())) for q in range(0, len(a2), bt)]
    clk_mhz = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("sm_max_mhz", 1965.0)) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 1965.0
    floor_ms = 8.0 * sum(longest) / (clk_mhz * 1e3)
    w0 = np.zeros(4096)
    st2 = []
    for _ in range(5):
        t0 = time.perf_counter()
        ctx.sgd_epoch(f2, a2, b2, y2, bt, 0.1, 1.0, w0)
        st2.append(time.perf_counter() - t0)
    sgd_ms = 1e3 * float(np.median(st2[1:]))
    c2["sgd_epoch"] = {"ms": sgd_ms, "steps": len(longest), "floor_ms": floor_ms, "frac": floor_ms / sgd_ms,
                       "bound": "latency",
                       "floor_model": "sum over the %d steps of the step's longest score chain (%d entries) "
                                      "x 8 cycles (DADD latency) at the max SM clock; the gradient folds and "
                                      "barriers are not in the floor" % (len(longest), sum(longest)),
                       "api": "pars_sgd_epoch (cluster kernel; host weights in/out)"}
    f2.free()
    if have_ref:
        rd2 = R.synthesize(8192, 21)
        t0 = time.perf_counter()
        R.train(rd2, OEx.make(), seed=21, epochs=1)
        c2["cpu_epoch_ms"] = 1e3 * (time.perf_counter() - t0)
        c2["cpu_threads"] = thr
    out["c2"] = c2
    # ---- C3: 100k-request Poisson simulation, FCFS vs PARS (C1 model), the
    # reference's own driver linked with the drop-in vs with the reference
    c3b, c3r = ROOT / "oracle" / "_ref" / "c3_b200", ROOT / "oracle" / "_ref" / "c3_ref"
    if c3b.exists():
        import subprocess
        env = dict(os.environ, OMP_NUM_THREADS="1")
        rb = json.loads(subprocess.run([str(c3b)], capture_output=True, text=True, env=env,
                                       timeout=900).stdout.strip().splitlines()[-1])
        c3 = {"workload": "run_simulation of 100,000 Poisson requests (5 req/s, batch 32) with "
                          "FCFS and PARS (README model) priorities; tools/c3_main.cpp linked with "
                          "the drop-in (GPU-scored priorities, incremental queue)",
              "gpu_pars_sim_s": rb["pars"]["wall_s"], "gpu_fcfs_sim_s": rb["fcfs"]["wall_s"],
              "pars_completion_fnv": rb["pars"]["completion_fnv"],
              "fcfs_completion_fnv": rb["fcfs"]["completion_fnv"],
              "parity_bitexact": rb["pars"]["completion_fnv"] == "322bc376a55e1141"
              and rb["fcfs"]["completion_fnv"] == "7be6c188801b08ca"}
        if have_ref and c3r.exists():
            rr = json.loads(subprocess.run([str(c3r)], capture_output=True, text=True, env=env,
                                           timeout=900).stdout.strip().splitlines()[-1])
            c3["cpu_pars_sim_s"] = rr["pars"]["wall_s"]
            c3["cpu_fcfs_sim_s"] = rr["fcfs"]["wall_s"]
            c3["cpu_threads"] = 1
        out["c3"] = c3
    # ---- C5, CPU side: all-pairs mask + hinge over a bounded sample
    if have_ref:
        O = Oracle()
        nS = 16384
        wl = P.Workload.synthesize(nS, 25)
        s = np.random.default_rng(99).normal(size=nS) * 0.05
        t0 = time.perf_counter()
        _, kept, _, _ = O.allpairs(s, wl.output_len, DELTA, MARGIN, threads=thr)
        dt = time.perf_counter() - t0
        out["c5_cpu"] = {"kind": "port", "sample": f"all pairs of the first {nS} C5-style prompts",
                         "filtered_pairs_per_s": kept / dt, "threads": thr}
    return out


def main():
    global N_PROMPTS
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=200000)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-pairs", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
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
