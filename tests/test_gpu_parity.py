"""GPU parity: every CUDA path through the C ABI against the oracle / the
reference's golden fixtures. Bit-exact for features, exact-mode scores,
masks, coefficients, counts, orders and the SGD trajectory; fast fp32 mode
within 1e-5 of sum|w_i v_i| (the magnitude scale)."""
import os

import numpy as np
import pytest

from conftest import extractor_from, golden, unhex
from oracle.bind import Extractor as OEx
from oracle.bind import fnv64_array

pytestmark = pytest.mark.gpu


def oex(e):
    return OEx.make(dim=e.dim, word=tuple(e.word[:e.n_word]), char=tuple(e.chr[:e.n_char]),
                    norm="l2" if e.norm else "none", kind="hashed" if e.kind == 0 else "embedding")


def grouped_feature_cases():
    groups = {}
    for c in golden("features.json")["cases"]:
        key = repr(c["extractor"])
        groups.setdefault(key, (c["extractor"], []))[1].append(c)
    return list(groups.values())


@pytest.mark.parametrize("desc,cases", grouped_feature_cases(),
                         ids=lambda v: str(v.get("dim")) if isinstance(v, dict) else "")
def test_extract_matches_reference_goldens(ctx, desc, cases):
    from paper_2510_03243_b200 import pack_texts
    e = extractor_from(desc)
    texts = [bytes.fromhex(c["text"]) for c in cases]
    # prefix the arena so offsets[0] != 0 and prompt starts are unaligned
    arena, offs = pack_texts([b"#pad#"] + texts)
    feats = ctx.extract(e, arena, offs[1:])
    rp, idx, val = feats.download()
    for k, c in enumerate(cases):
        got_i = idx[rp[k]:rp[k + 1]]
        got_v = val[rp[k]:rp[k + 1]]
        assert got_i.tolist() == c["idx"], (k, c["text"][:40])
        assert [float(v).hex() for v in got_v] == c["val"], (k, c["text"][:40])


@pytest.mark.parametrize("desc,cases", grouped_feature_cases(),
                         ids=lambda v: str(v.get("dim")) if isinstance(v, dict) else "")
def test_exact_scores_bit_identical(ctx, oracle, desc, cases):
    from paper_2510_03243_b200 import MODE_EXACT, pack_texts
    e = extractor_from(desc)
    texts = [bytes.fromhex(c["text"]) for c in cases]
    rng = np.random.default_rng(desc["dim"])
    w = rng.normal(size=desc["dim"])
    arena, offs = pack_texts(texts)
    got = ctx.score_text(e, arena, offs, w, bias=0.125, mode=MODE_EXACT)
    want = oracle.score_batch(oex(e), arena, offs, w, 0.125)
    assert [x.hex() for x in got] == [x.hex() for x in want]


def test_fast_scores_within_tolerance(ctx, oracle):
    from paper_2510_03243_b200 import MODE_FAST, Workload
    wl = Workload.synthesize(3000, 5)
    e = extractor_from(dict(kind=0, dim=4096, norm=1, word=[1], char=[3]))
    w = np.random.default_rng(0).normal(size=4096)
    got = ctx.score_text(e, wl.text, wl.offsets, w, 0.5, mode=MODE_FAST)
    want = oracle.score_batch(oex(e), wl.text, wl.offsets, w, 0.5)
    # magnitude scale sum |w_i v_i| per prompt
    rp, idx, val = oracle.extract_all(oex(e), wl.text, wl.offsets)
    scale = np.array([np.abs(w[idx[rp[i]:rp[i + 1]]] * val[rp[i]:rp[i + 1]]).sum() + 0.5
                      for i in range(len(wl))])
    rel = np.abs(got - want) / scale
    assert rel.max() <= 1e-5, rel.max()


def test_long_prompts_take_the_wide_counter_path(ctx, oracle):
    from paper_2510_03243_b200 import MODE_EXACT, pack_texts
    e = extractor_from(dict(kind=0, dim=4096, norm=1, word=[1], char=[3]))
    long1 = b" ".join(b"tok%d" % (i % 17) for i in range(20000))  # >32767 features
    long2 = b"aaa " * 40000  # one bucket with a count far above 2^15
    texts = [b"short one", long1, b"x", long2, b""]
    arena, offs = pack_texts(texts)
    w = np.random.default_rng(2).normal(size=4096)
    got = ctx.score_text(e, arena, offs, w, 0.0, MODE_EXACT)
    want = oracle.score_batch(oex(e), arena, offs, w, 0.0)
    assert [x.hex() for x in got] == [x.hex() for x in want]
    f = ctx.extract(e, arena, offs)
    rp, idx, val = f.download()
    orp, oidx, oval = oracle.extract_all(oex(e), arena, offs)
    assert (rp == orp).all() and (idx == oidx).all() and (val == oval).all()


def test_readme_workload_scores_and_sjf_order(ctx):
    """Appendix B: gen(500, seed 22) scored with the README model; burst
    SJF order FNV 7432e2f4c44cbabd."""
    from paper_2510_03243_b200 import Extractor, Workload, tie_ranks
    m = golden("models.json")
    z = golden("readme_model.npz")
    w = z["weights"]
    assert fnv64_array(w) == m["readme"]["weights_fnv"]
    wl = Workload.synthesize(500, 22)
    s = ctx.score_text(Extractor.make(), wl.text, wl.offsets, w)
    assert [x.hex() for x in s] == [x.hex() for x in z["s500"]]
    ids = ["p%06d" % i for i in range(500)]
    order = ctx.priority_order(s, tie_ranks(np.zeros(500), ids))
    assert fnv64_array(order.astype(np.uint64)) == m["workload500"]["order_fnv"]


def test_c1_scores_and_order(ctx):
    """Config 1: 1,024 prompts (<=128 tokens) scored and sorted, bit-exact."""
    from paper_2510_03243_b200 import Extractor, Workload, tie_ranks
    m = golden("models.json")
    z = golden("readme_model.npz")
    g = Workload.synthesize(2048, 22)
    sel = z["c1_index"]
    texts = [g.prompt(i) for i in sel]
    from paper_2510_03243_b200 import pack_texts
    arena, offs = pack_texts(texts)
    s = ctx.score_text(Extractor.make(), arena, offs, z["weights"])
    assert fnv64_array(s) == m["c1"]["scores_fnv"] == "5548c3b3d81d615d"
    ids = ["p%06d" % i for i in sel]
    order = ctx.priority_order(s, tie_ranks(np.zeros(len(sel)), ids))
    assert fnv64_array(order.astype(np.uint64)) == m["c1"]["order_fnv"] == "e6e78f54425df769"


def test_priority_order_matches_select_batch_goldens(ctx):
    from paper_2510_03243_b200 import tie_ranks
    for c in golden("select.json"):
        arrival, score = unhex(c["arrival"]), unhex(c["score"])
        order = ctx.priority_order(score, tie_ranks(arrival, c["ids"]), np.array(c["boosted"], np.uint8))
        assert order.tolist() == c["order"]


def test_priority_order_large_random_with_ties(ctx, oracle):
    from paper_2510_03243_b200 import tie_ranks
    rng = np.random.default_rng(7)
    n = 200_000
    score = rng.choice(np.concatenate([rng.normal(size=50), [0.0, -0.0]]), size=n)
    arrival = rng.choice(np.arange(100) * 0.25, size=n)
    ids = ["q%d" % rng.integers(0, 1000) for _ in range(n)]
    boosted = (rng.random(n) < 0.05).astype(np.uint8)
    got = ctx.priority_order(score, tie_ranks(arrival, ids), boosted)
    want = oracle.select_order(arrival, ids, score, boosted, 1e9)
    assert (got == want).all()


@pytest.mark.parametrize("algo", ["sorted", "general"])
def test_allpairs_matches_oracle(ctx, oracle, algo):
    rng = np.random.default_rng(3)
    for n in (1, 2, 255, 256, 257, 3001):
        lens = rng.integers(1, 400, size=n)
        s = rng.normal(size=n)
        c, kept, act, loss = ctx.allpairs(s, lens, 0.2, 1.0, algo=algo)
        oc, okept, oact, oloss = oracle.allpairs(s, lens, 0.2, 1.0)
        assert (c == oc).all() and kept == okept and act == oact
        assert abs(loss - oloss) <= 1e-12 * max(1.0, abs(oloss))


@pytest.mark.parametrize("algo", ["sorted", "general"])
def test_allpairs_hinge_edge_cases(ctx, oracle, algo):
    """Ties in scores and lengths, +-0.0, scores exactly margin apart, tiny
    and huge magnitudes, margin 0: the active set must match bit-exactly."""
    rng = np.random.default_rng(11)
    n = 1500
    base = np.array([0.0, -0.0, 1.0, -1.0, 0.5, 1e-300, -1e-300, 3.0, 2.0, 1e15, -1e15,
                     0.1, 0.2, 0.30000000000000004, np.nextafter(1.0, 2.0)])
    s = rng.choice(base, size=n) + rng.choice([0.0, 1.0, -1.0], size=n)
    lens = rng.choice([1, 2, 3, 5, 8, 10, 12, 50, 51, 60, 1000], size=n)
    for margin in (1.0, 0.0, 0.5):
        for delta in (0.2, 0.0, 0.5):
            c, kept, act, loss = ctx.allpairs(s, lens, delta, margin, algo=algo)
            oc, okept, oact, oloss = oracle.allpairs(s, lens, delta, margin)
            assert (c == oc).all() and kept == okept and act == oact, (margin, delta)
            assert abs(loss - oloss) <= 1e-9 * max(1.0, abs(oloss))


def test_pair_plan_kept_counts_match_exhaustive_goldens(ctx):
    """The plan's exact kept count equals the exhaustive Eq. 1 counts of
    SURVEY Appendix B (C2: 30,028,032; C5: 1,920,977,782)."""
    from paper_2510_03243_b200 import Workload
    g = golden("mask_counts.json")
    for key in ("8192_21", "65536_25", "1024_22"):
        e = g[key]
        wl = Workload.synthesize(e["n"], e["seed"], mu=e["mu"], sigma=e["sigma"])
        plan = ctx.pair_plan(wl.output_len, e["delta"])
        assert plan.sorted and plan.kept == e["kept"]


def test_allpairs_c2_mask_count(ctx):
    """C2 dataset: exhaustive Eq. 1 count 30,028,032;
    at w = 0 every kept pair is active with loss exactly margin."""
    from paper_2510_03243_b200 import Workload
    wl = Workload.synthesize(8192, 21)
    c, kept, act, loss = ctx.allpairs(np.zeros(8192), wl.output_len, 0.2, 1.0)
    assert kept == 30_028_032 == act
    assert loss == float(kept)


@pytest.mark.parametrize("algo", ["auto", "sorted", "pairs"])
def test_kendall_tau_matches_goldens_and_oracle(ctx, oracle, algo):
    for c in golden("tau.json"):
        tau, counts = ctx.kendall_tau(unhex(c["x"]), unhex(c["y"]), algo)
        assert counts.tolist() == c["counts"]
        assert float(tau).hex() == c["tau"]
    rng = np.random.default_rng(9)
    x = rng.integers(0, 50, size=5000).astype(float)
    y = rng.normal(size=5000).round(2)
    tau, counts = ctx.kendall_tau(x, y, algo)
    otau, ocounts = oracle.kendall(x, y)
    assert counts.tolist() == ocounts.tolist() and tau == otau


@pytest.mark.parametrize("n", [2, 3, 17, 2047, 2048, 2049, 4096, 6000, 30011])
def test_kendall_sorted_counts_exact(ctx, oracle, n):
    """The O(n log n) counts (tau_sorted.cu) equal the reference's all-pairs
    integers across tile boundaries (2,048), heavy ties in x, y and both,
    and signed zeros (-0.0 == +0.0 is a tie)."""
    rng = np.random.default_rng(n)
    for x, y in ((rng.normal(size=n), rng.normal(size=n)),
                 (rng.integers(0, 7, n).astype(float), rng.integers(0, 5, n).astype(float)),
                 (np.where(rng.random(n) < 0.4, 0.0, np.where(rng.random(n) < 0.5, -0.0, 1.0)),
                  rng.normal(size=n).round(1)),
                 (np.arange(n, dtype=float), -np.arange(n, dtype=float)),
                 (np.arange(n, dtype=float) % 3, np.arange(n, dtype=float))):
        if (x == x[0]).all() or (y == y[0]).all():
            continue
        otau, oc = oracle.kendall(x, y, threads=os.cpu_count() or 1)
        tau, c = ctx.kendall_tau(x, y, "sorted")
        assert c.tolist() == oc.tolist() and tau == otau


def test_kendall_sorted_graph_replay_and_recapture(ctx, oracle):
    """The sorted counts run as a CUDA graph cached on (inputs, n, scratch):
    new contents of the same device buffers replay it, a shorter n on the
    same pointers and a non-finite value (the tile path) re-check it; every
    call against the reference's all-pairs integers."""
    import torch
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(77)
    n = 5000
    dx = torch.empty(n, dtype=torch.float64, device=dev)
    dy = torch.empty(n, dtype=torch.float64, device=dev)
    cases = [(rng.normal(size=n), rng.integers(0, 40, n).astype(float), n),
             (rng.integers(0, 9, n).astype(float), rng.normal(size=n), n),
             (rng.normal(size=n), rng.normal(size=n).round(1), 2049),
             (rng.normal(size=n), rng.integers(0, 40, n).astype(float), n)]
    for x, y, m in cases:
        dx.copy_(torch.from_numpy(x))
        dy.copy_(torch.from_numpy(y))
        torch.cuda.synchronize()
        tau, c = ctx.dev_kendall_tau(dx.data_ptr(), dy.data_ptr(), m)
        otau, oc = oracle.kendall(x[:m], y[:m], threads=os.cpu_count() or 1)
        assert [int(v) for v in c] == oc.tolist() and tau == otau
    x[3] = np.inf
    dx.copy_(torch.from_numpy(x))
    torch.cuda.synchronize()
    tau, c = ctx.dev_kendall_tau(dx.data_ptr(), dy.data_ptr(), n)
    otau, oc = oracle.kendall(x, y, threads=os.cpu_count() or 1)
    assert [int(v) for v in c] == oc.tolist() and tau == otau


def test_kendall_non_finite_falls_back_to_pairs(ctx, oracle):
    """inf - inf = NaN is neither a tie nor negative in the reference, so the
    sorted method does not apply: auto runs the all-pairs tiles."""
    from paper_2510_03243_b200 import ParsError
    rng = np.random.default_rng(4)
    x = rng.normal(size=3000)
    y = rng.normal(size=3000)
    x[[5, 9, 700]] = [np.inf, np.inf, -np.inf]
    y[[11, 12]] = [np.nan, np.inf]
    otau, oc = oracle.kendall(x, y)
    tau, c = ctx.kendall_tau(x, y, "auto")
    assert c.tolist() == oc.tolist() and tau == otau
    with pytest.raises(ParsError, match="finite"):
        ctx.kendall_tau(x, y, "sorted")


def test_kendall_sorted_large_matches_pairs(ctx):
    """At the C3 trace size both GPU algorithms give the same integers."""
    import torch
    from paper_2510_03243_b200 import Workload
    wl = Workload.synthesize(100_000, 23)
    x = np.random.default_rng(1).normal(size=100_000).round(3)
    y = wl.output_len.astype(np.float64)
    t1, c1 = ctx.kendall_tau(x, y, "sorted")
    t2, c2 = ctx.kendall_tau(x, y, "pairs")
    assert c1.tolist() == c2.tolist() and t1 == t2
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    t3, c3 = ctx.dev_kendall_tau(dx.data_ptr(), dy.data_ptr(), len(x))
    assert c3.tolist() == c1.tolist() and t3 == t1


def test_kendall_degenerate_error(ctx):
    from paper_2510_03243_b200 import ParsError
    with pytest.raises(ParsError, match="degenerate ranking"):
        ctx.kendall_tau(np.ones(10), np.arange(10.0))


@pytest.mark.parametrize("algo", ["cluster", "single"])
def test_sgd_epoch_bit_identical(ctx, oracle, algo):
    from paper_2510_03243_b200 import Extractor, Workload, build_pairs
    wl = Workload.synthesize(1500, 12)
    e = Extractor.make()
    f = ctx.extract(e, wl.text, wl.offsets)
    rp, idx, val = f.download()
    a, b, y, _ = build_pairs(wl.output_len, 0.2, 20000, 99)
    w0 = np.random.default_rng(1).normal(size=4096) * 0.01
    for batch in ((128, 1, 7, 4096) if algo == "single" else (128, 1, 7, 96, 200)):
        w, el, act = ctx.sgd_epoch(f, a, b, y, batch, 0.1, 1.0, w0, algo=algo)
        ow, oel, oact = oracle.sgd_epoch(rp, idx, val, 4096, a, b, y, batch, 0.1, 1.0, w0)
        assert act == oact
        assert el.hex() == oel.hex()
        assert (w.view(np.uint64) == ow.view(np.uint64)).all()


def test_train_small_goldens(ctx):
    from paper_2510_03243_b200 import Extractor, Workload
    for c in golden("train_small.json"):
        wl = Workload.synthesize(c["n"], c["seed"])
        w, b, lt = ctx.train_pairwise(Extractor.make(dim=c["dim"]), wl.text, wl.offsets,
                                      wl.output_len, delta=c["delta"], margin=c["margin"],
                                      epochs=c["epochs"], batch=c["batch"], lr=c["lr"],
                                      seed=c["seed"], pairs_per_epoch=c["ppe"])
        assert [float(x).hex() for x in lt] == c["loss_trace"]
        assert fnv64_array(w) == c["weights_fnv"]


def test_readme_training_pipeline_bit_identical(ctx, ref):
    """README recipe (gen 4000 seed 21, split 0.2, train seed 21): weights
    FNV db7217cbd5a86b9b and the loss trace, trained on the GPU."""
    from paper_2510_03243_b200 import Extractor
    m = golden("models.json")
    full = ref.synthesize(4000, 21)
    tr, _ = ref.split(full, 0.2, 21)
    w, b, lt = ctx.train_pairwise(Extractor.make(), tr.text, tr.offs, tr.output_len, seed=21)
    assert fnv64_array(w) == m["readme"]["weights_fnv"]
    assert [float(x).hex() for x in lt] == m["readme"]["loss_trace"]


def test_c2_epoch_bit_identical(ctx):
    """Config 2: one epoch on gen(8192, seed 21): loss 0.55296763305525443,
    weights FNV f97c96a353829ee2."""
    from paper_2510_03243_b200 import Extractor, Workload
    m = golden("models.json")
    wl = Workload.synthesize(8192, 21)
    w, b, lt = ctx.train_pairwise(Extractor.make(), wl.text, wl.offsets, wl.output_len, seed=21,
                                  epochs=1)
    assert float(lt[0]).hex() == m["c2"]["loss0"]
    assert fnv64_array(w) == m["c2"]["weights_fnv"] == "f97c96a353829ee2"


@pytest.mark.parametrize("n,dim", [(300, 64), (1000, 100), (129, 7), (1, 4096), (600, 4096), (513, 34), (300, 2)])
def test_embedding_scores_exact(ctx, oracle, n, dim):
    """Cooperative dense kernel: row-block tails (n % 256), column-tile tails
    (dim % 32), odd dims (the simple kernel), fast mode within 1e-5."""
    from paper_2510_03243_b200 import MODE_EXACT, MODE_FAST, Extractor
    rng = np.random.default_rng(4)
    for norm in ("l2", "none"):
        e = Extractor.make(dim=dim, kind="embedding", norm=norm)
        X = rng.normal(size=(n, dim))
        X[0] = 0.0
        w = rng.normal(size=dim)
        got = ctx.score_embeddings(e, X, w, 0.25, MODE_EXACT)
        want = oracle.score_dense(oex(e), X, w, 0.25)
        assert [x.hex() for x in got] == [x.hex() for x in want]
        fast = ctx.score_embeddings(e, X, w, 0.25, MODE_FAST)
        nrm = np.sqrt((X * X).sum(1, keepdims=True)) if norm == "l2" else 1.0
        V = X / np.where(nrm > 0, nrm, 1.0)
        scale = np.abs(V * w).sum(1) + 0.25  # sum |w_i v_i| + |bias|
        assert (np.abs(fast - want) / scale).max() <= 1e-5


def test_features_score_matches_linear_scorer(ctx, oracle):
    from paper_2510_03243_b200 import Extractor, Workload
    wl = Workload.synthesize(700, 8)
    e = Extractor.make()
    f = ctx.extract(e, wl.text, wl.offsets)
    w = np.random.default_rng(5).normal(size=4096)
    got = f.score(w, -0.5)
    want = oracle.score_batch(oex(e), wl.text, wl.offsets, w, -0.5)
    assert [x.hex() for x in got] == [x.hex() for x in want]


def test_errors_are_loud(ctx):
    from paper_2510_03243_b200 import Extractor, ParsError, pack_texts
    arena, offs = pack_texts([b"a b"])
    with pytest.raises(ParsError, match="feature extractor dimension is 0"):
        ctx.score_text(Extractor.make(dim=0), arena, offs, np.zeros(1))
    with pytest.raises(ParsError, match="word n-gram order must be >= 1"):
        ctx.score_text(Extractor.make(word=(0,)), arena, offs, np.zeros(4096))
    with pytest.raises(ParsError, match=r"train: delta 1 outside \[0, 1\)"):
        ctx.train_pairwise(Extractor.make(), arena, offs, np.array([3]), delta=1.0)


def test_distributed_allpairs_step_single_rank(ctx, oracle):
    """distributed.allpairs_step_gpu (the C5 exchange step) on one rank equals
    the all-pairs oracle; grad_step_gpu equals X^T c."""
    import torch
    from paper_2510_03243_b200 import Extractor, Workload
    from paper_2510_03243_b200 import distributed as D
    wl = Workload.synthesize(3000, 41)
    e = Extractor.make()
    w = np.random.default_rng(6).normal(size=4096) * 0.1
    s = ctx.score_text(e, wl.text, wl.offsets, w)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        d_s = torch.from_numpy(s).to(dev)
        d_L = torch.from_numpy(wl.output_len.astype(np.int32)).to(dev)
        plan = ctx.pair_plan(wl.output_len, 0.2)
        c, kept, act, loss = D.allpairs_step_gpu(ctx, d_s, d_L, len(s), 0.2, 1.0,
                                                 int(wl.output_len.max()), stream=stream.cuda_stream,
                                                 plan=plan)
        c2, kept2, act2, loss2 = D.allpairs_step_gpu(ctx, d_s, d_L, len(s), 0.2, 1.0,
                                                     int(wl.output_len.max()),
                                                     stream=stream.cuda_stream)
        assert (c2.cpu().numpy() == c.cpu().numpy()).all() and (kept2, act2) == (kept, act)
        oc, okept, oact, oloss = oracle.allpairs(s, wl.output_len, 0.2, 1.0)
        assert (c.cpu().numpy() == oc).all() and kept == okept and act == oact
        assert abs(loss - oloss) <= 1e-12 * max(1.0, oloss)
        f = ctx.extract(e, wl.text, wl.offsets)
        g = D.grad_step_gpu(ctx, f, c, 1.0, stream=stream.cuda_stream).cpu().numpy()
    rp, idx, val = f.download()
    og = oracle.xt_c(rp, idx, val, oc, 4096)
    assert np.allclose(g, og, rtol=1e-12, atol=1e-12)


def test_sgd_cluster_long_prompts_use_global_fallback(ctx, oracle):
    """Rows too large for the staged buffers (2,048-token prompts) are read
    from global memory by the cluster kernel: still bit-identical."""
    from paper_2510_03243_b200 import Extractor, Workload, build_pairs
    wl = Workload.synthesize(300, 14, pad_tokens=2048, pad_seed=3)
    e = Extractor.make()
    f = ctx.extract(e, wl.text, wl.offsets)
    rp, idx, val = f.download()
    a, b, y, _ = build_pairs(wl.output_len, 0.2, 3000, 5)
    w0 = np.random.default_rng(2).normal(size=4096) * 0.01
    w, el, act = ctx.sgd_epoch(f, a, b, y, 128, 0.1, 1.0, w0, algo="cluster")
    ow, oel, oact = oracle.sgd_epoch(rp, idx, val, 4096, a, b, y, 128, 0.1, 1.0, w0)
    assert act == oact and el.hex() == oel.hex()
    assert (w.view(np.uint64) == ow.view(np.uint64)).all()


def _random_texts(n, seed):
    rng = np.random.default_rng(seed)
    alpha = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz0123456789  \t\n\v\f\r\x80\xc3\xa9\xff\x1f", np.uint8)
    out = []
    for k in range(n):
        L = int(rng.choice([0, 1, 2, 3, 4, 5, 7, 31, 32, 33, 64, 127, 128, 129, 500, 2170, 5000]))
        t = alpha[rng.integers(0, len(alpha), L)].tobytes()
        if k % 7 == 0 and L > 10:  # a long token across several lane ranges
            t = t[:3] + b"q" * (L // 2) + t[3 + L // 2:]
        out.append(t)
    return out


@pytest.mark.parametrize("dim", [512, 1024, 4096, 16384])
def test_sequential_lane_kernel_random_texts(ctx, oracle, dim):
    """Ragged prompts (empty, 1-byte, lane-boundary lengths, every C-locale
    space, bytes >= 0x80, tokens spanning many lane ranges) at unaligned
    offsets: exact scores and CSR rows bit-identical, fast mode in tolerance.
    dim 512 exercises the general kernel, the rest the sequential-lane one."""
    from paper_2510_03243_b200 import MODE_EXACT, MODE_FAST, pack_texts
    e = extractor_from(dict(kind=0, dim=dim, norm=1, word=[1], char=[3]))
    texts = _random_texts(600, dim)
    arena, offs = pack_texts([b"##"] + texts)
    offs = offs[1:]
    w = np.random.default_rng(dim + 1).normal(size=dim)
    got = ctx.score_text(e, arena, offs, w, -0.25, MODE_EXACT)
    want = oracle.score_batch(oex(e), arena, offs, w, -0.25)
    assert (got.view(np.uint64) == want.view(np.uint64)).all()
    f = ctx.extract(e, arena, offs)
    rp, idx, val = f.download()
    orp, oidx, oval = oracle.extract_all(oex(e), arena, offs)
    assert (rp == orp).all() and (idx == oidx).all() and (val.view(np.uint64) == oval.view(np.uint64)).all()
    fast = ctx.score_text(e, arena, offs, w, -0.25, MODE_FAST)
    scale = np.array([np.abs(w[oidx[orp[i]:orp[i + 1]]] * oval[orp[i]:orp[i + 1]]).sum() + 0.25
                      for i in range(len(texts))])
    assert (np.abs(fast - want) / scale).max() <= 1e-5


@pytest.mark.parametrize("n", [1, 2, 3, 31, 1000, 1024, 4095, 4096, 4097, 9000])
def test_priority_order_sizes(ctx, oracle, n):
    """The single-CTA bitonic path (n <= 4096) and the radix path on either
    side of the switch: ties in score and (arrival, id), -0.0 vs +0.0, boosts."""
    from paper_2510_03243_b200 import tie_ranks
    rng = np.random.default_rng(n)
    score = rng.choice(np.concatenate([rng.normal(size=7), [0.0, -0.0]]), size=n)
    arrival = rng.choice(np.arange(5) * 0.5, size=n)
    ids = ["r%d" % rng.integers(0, 9) for _ in range(n)]
    boosted = (rng.random(n) < 0.1).astype(np.uint8)
    got = ctx.priority_order(score, tie_ranks(arrival, ids), boosted)
    want = oracle.select_order(arrival, ids, score, boosted, 1e9)
    assert (got == want).all()


def test_score_order_fused_matches_two_calls_and_oracle(ctx, oracle):
    """pars_score_order == pars_score_text + pars_priority_order == the
    reference's score_batch + select_batch (C1-shaped: 1,024 prompts)."""
    from paper_2510_03243_b200 import Extractor, Workload, tie_ranks
    wl = Workload.synthesize(1024, 22)
    w = golden("readme_model.npz")["weights"]
    ids = ["p%06d" % i for i in range(len(wl))]
    arrival = np.zeros(len(wl))
    tie = tie_ranks(arrival, ids)
    boosted = (np.arange(len(wl)) % 97 == 0).astype(np.uint8)
    s, order = ctx.score_order(Extractor.make(), wl.text, wl.offsets, w, tie, boosted)
    s2 = ctx.score_text(Extractor.make(), wl.text, wl.offsets, w)
    assert (s.view(np.uint64) == s2.view(np.uint64)).all()
    assert (order == ctx.priority_order(s2, tie, boosted)).all()
    assert (order == oracle.select_order(arrival, ids, s2, boosted, 0.0)).all()


@pytest.mark.parametrize("n", [1, 3000, 300_000])
def test_score_order_into_pinned_buffers(ctx, n):
    """Page-locked caller buffers take the scores and the order by direct DMA
    (no staging); results equal the pageable-buffer call, across chunk
    boundaries of the host pipeline (300k prompts = several chunks)."""
    from paper_2510_03243_b200 import Extractor, Workload, pinned_empty
    wl = Workload.synthesize(n, 5)
    w = np.random.default_rng(2).normal(size=4096) * 0.05
    tie = np.arange(n, dtype=np.uint32)[::-1].copy()
    s1, o1 = ctx.score_order(Extractor.make(), wl.text, wl.offsets, w, tie)
    outs = (pinned_empty(n, np.float64), pinned_empty(n, np.int64))
    outs[0][:] = np.nan
    s3 = ctx.score_text(Extractor.make(), wl.text, wl.offsets, w, out=outs[0])
    assert (s3.view(np.uint64) == s1.view(np.uint64)).all()
    for _ in range(2):  # reused buffers
        outs[0][:] = np.nan
        outs[1][:] = -1
        s2, o2 = ctx.score_order(Extractor.make(), wl.text, wl.offsets, w, tie, out=outs)
        assert (s2.view(np.uint64) == s1.view(np.uint64)).all()
        assert (o2 == o1).all()


def test_dev_features_score_compact_rows_bit_identical(ctx, oracle):
    """pars_dev_features_score (the scoring step of the DP training step)
    over the compact (idx, count16) rows, row shards included, equals the
    reference's score_batch bit for bit."""
    import ctypes
    import torch
    from paper_2510_03243_b200 import Extractor, Workload, lib
    wl = Workload.synthesize(2500, 12)
    e = Extractor.make()
    f = ctx.extract(e, wl.text, wl.offsets)
    w = np.random.default_rng(13).normal(size=4096)
    d_w = torch.from_numpy(w).cuda()
    out = torch.full((len(wl),), float("nan"), dtype=torch.float64, device="cuda")
    for r0, r1 in ((0, 1000), (1000, 1001), (1001, len(wl))):
        assert lib().pars_dev_features_score(ctx.h, ctypes.c_void_p(f.h), r0, r1, d_w.data_ptr(), 0.5,
                                             out.data_ptr(), None) == 0
    torch.cuda.synchronize()
    want = oracle.score_batch(oex(e), wl.text, wl.offsets, w, 0.5)
    assert (out.cpu().numpy().view(np.uint64) == want.view(np.uint64)).all()
    f.free()


def test_kendall_tau_tile_split_matches_single_call(ctx, oracle):
    """pars_dev_kendall_counts over tile slices (as data-parallel ranks would
    run them) sums to pars_kendall_tau's counts; the finish is finish_tau."""
    import torch
    from paper_2510_03243_b200 import distributed as D
    rng = np.random.default_rng(8)
    n = 3001
    x = rng.integers(0, 100, n).astype(np.float64)
    y = x * 0.5 + rng.integers(0, 60, n)
    tau1, c1 = ctx.kendall_tau(x, y)
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    tau2, c2 = D.kendall_tau_gpu(ctx, dx, dy, n)
    assert tau1 == tau2 and (c1 == c2).all()
    otau, oc = oracle.kendall(x, y)
    assert (c2 == oc).all() and tau2 == otau


def test_weights_upload_cache_is_invalidated(ctx):
    """Host-buffer calls skip re-uploading unchanged weights; the cache must
    follow every change (new weights, other device weights through the
    pars_dev_* paths, fp32 conversions)."""
    import torch
    from paper_2510_03243_b200 import MODE_EXACT, MODE_FAST, Extractor, Workload
    wl = Workload.synthesize(700, 3)
    ex = Extractor.make()
    rng = np.random.default_rng(8)
    w1, w2 = rng.normal(size=4096), rng.normal(size=4096)
    ref = {}
    for name, w in (("w1", w1), ("w2", w2)):
        for mode in (MODE_EXACT, MODE_FAST):
            other = Context_fresh(ctx)
            ref[name, mode] = other.score_text(ex, wl.text, wl.offsets, w, mode=mode)
    seq = [("w1", MODE_EXACT), ("w1", MODE_FAST), ("w1", MODE_EXACT), ("w2", MODE_FAST),
           ("w2", MODE_EXACT), ("w1", MODE_FAST), ("w1", MODE_FAST)]
    d_text = torch.from_numpy(wl.text).cuda()
    d_offs = torch.from_numpy(wl.offsets).cuda()
    d_w2 = torch.from_numpy(w2).cuda()
    d_out = torch.empty(len(wl), dtype=torch.float64, device="cuda")
    for name, mode in seq:
        w = w1 if name == "w1" else w2
        got = ctx.score_text(ex, wl.text, wl.offsets, w.copy(), mode=mode)
        assert (got.view(np.uint64) == ref[name, mode].view(np.uint64)).all(), (name, mode)
        # device-weight scoring in fast mode overwrites the fp32 weight buffer
        ctx.dev_score_text(ex, d_text.data_ptr(), d_offs.data_ptr(), len(wl), d_w2.data_ptr(), 0.0,
                           MODE_FAST, d_out.data_ptr())
        torch.cuda.synchronize()


def Context_fresh(ctx):
    from paper_2510_03243_b200 import Context
    return Context(0)


@pytest.mark.parametrize("n,runs", [(1, 1), (1000, 2), (300_001, 4), (1_000_003, 8), (77, 3),
                                    (4096, 5)])
def test_merge_shard_orders_equals_global_order(ctx, n, runs):
    """pars_dev_merge_orders: the select_batch order of all prompts from the
    orders of contiguous shards equals one pars_dev_priority_order over all —
    with equal scores, boosted prompts and repeated tie ranks."""
    import ctypes
    import torch
    from paper_2510_03243_b200 import lib
    rng = np.random.default_rng(n + runs)
    s = rng.normal(size=n).round(2)  # many equal scores
    s[rng.random(n) < 0.01] = -0.0
    tie = rng.integers(0, max(1, n // 3), n).astype(np.uint32)
    boosted = (rng.random(n) < 0.05).astype(np.uint8)
    ds, dt, db = (torch.from_numpy(s).cuda(), torch.from_numpy(tie).cuda(),
                  torch.from_numpy(boosted).cuda())
    want = torch.empty(n, dtype=torch.int32, device="cuda")
    assert lib().pars_dev_priority_order(ctx.h, ds.data_ptr(), db.data_ptr(), dt.data_ptr(), n,
                                         want.data_ptr(), None) == 0
    offs = np.linspace(0, n, runs + 1).astype(np.int64)
    run_orders = torch.empty(n, dtype=torch.int32, device="cuda")
    for r in range(runs):
        a, b = int(offs[r]), int(offs[r + 1])
        if b > a:
            assert lib().pars_dev_priority_order(ctx.h, ds[a:].data_ptr(), db[a:].data_ptr(),
                                                 dt[a:].data_ptr(), b - a,
                                                 run_orders[a:].data_ptr(), None) == 0
    got = torch.empty(n, dtype=torch.int32, device="cuda")
    assert lib().pars_dev_merge_orders(ctx.h, ds.data_ptr(), db.data_ptr(), dt.data_ptr(),
                                       run_orders.data_ptr(), offs.ctypes.data, runs,
                                       got.data_ptr(), None) == 0
    torch.cuda.synchronize()
    assert (got.cpu().numpy() == want.cpu().numpy()).all()


def test_priority_order_graph_replay_follows_the_data(ctx):
    """pars_dev_priority_order captured once as a CUDA graph (its pass plan,
    the high-word speculation and the fallback gate are all decided on the
    device, its kernels chained by programmatic dependent launch) and replayed
    over new key contents: spread scores (the fixup holds), scores repeated
    40 times (no speculation), distinct scores on four top words (the fixup
    falls back to the full LSD) — each replay's order equal to lexsort."""
    import torch
    from paper_2510_03243_b200 import lib
    n = 300_000
    rng = np.random.default_rng(77)
    base = rng.normal(size=n) * 0.3
    inputs = [base,
              rng.choice(base[: n // 40], size=n),
              (1.0 + rng.integers(0, 2**32, size=n) * 2.0**-52) * rng.choice([1.0, 2.0, 4.0, 8.0], size=n)]
    tie = rng.integers(0, 1000, size=n).astype(np.uint32)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        d_s = torch.from_numpy(inputs[0]).to(dev)
        d_t = torch.from_numpy(tie.astype(np.int32)).to(dev)
        d_o = torch.empty(n, dtype=torch.int32, device=dev)

        def run():
            assert lib().pars_dev_priority_order(ctx.h, d_s.data_ptr(), None, d_t.data_ptr(), n,
                                                 d_o.data_ptr(), stream.cuda_stream) == 0
        run()  # scratch sized before capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            run()
        for s in inputs + inputs[::-1]:
            d_s.copy_(torch.from_numpy(s).to(dev))
            g.replay()
            torch.cuda.synchronize()
            want = np.lexsort((np.arange(n), tie, s))
            assert (d_o.cpu().numpy() == want).all()


def test_dp_train_step_replays_as_a_cuda_graph(ctx):
    """The C5 step (score, all-pairs plan tiles, X^T c, update) captured once as
    a CUDA graph and replayed trains bit-identically to launching it."""
    import torch
    from paper_2510_03243_b200 import Extractor, Workload
    from paper_2510_03243_b200 import distributed as D
    n = 4000
    wl = Workload.synthesize(n, 43)
    f = ctx.extract(Extractor.make(), wl.text, wl.offsets)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    w0 = np.random.default_rng(3).normal(size=4096) * 0.05
    with torch.cuda.stream(stream):
        d_w = torch.from_numpy(w0).to(dev)
        d_L = torch.from_numpy(wl.output_len.astype(np.int32)).to(dev)
        scores = torch.zeros(n, dtype=torch.float64, device=dev)
        plan = ctx.pair_plan(wl.output_len, 0.2)
        sh = stream.cuda_stream
        max_len = int(wl.output_len.max())

        def step():
            D.train_step_gpu(ctx, f, d_w, scores, d_L, n, 0.2, 1.0, max_len, 0.1 / plan.kept,
                             stream=sh, plan=plan)

        for _ in range(2):
            step()  # warm-up: lazily built structures exist before capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            step()
        d_w.copy_(torch.from_numpy(w0).to(dev))
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        w_graph = d_w.clone()
        d_w.copy_(torch.from_numpy(w0).to(dev))
        for _ in range(3):
            step()
        torch.cuda.synchronize()
    assert torch.equal(w_graph.view(torch.int64), d_w.view(torch.int64))
    assert not torch.equal(d_w, torch.from_numpy(w0).to(dev))
    f.free()


@pytest.mark.gpu
def test_score_records_gather_equals_score_text(ctx, oracle):
    """pars_score_records (records as separate host strings, gathered into
    pinned staging by host threads, several chunks) is bit-identical to
    pars_score_text over the packed arena and to the oracle."""
    from oracle.bind import Extractor as OEx
    from paper_2510_03243_b200 import Extractor, Workload
    wl = Workload.synthesize(40000, 22, pad_tokens=300)  # > 1 chunk of the 4 MB ramp
    texts = [wl.prompt(i) for i in range(len(wl))]
    texts[7] = b""  # an empty record
    w = np.random.default_rng(4).normal(size=4096)
    s = ctx.score_records(Extractor.make(), texts, w, 0.25)
    arena = np.frombuffer(b"".join(texts), np.uint8)
    offs = np.zeros(len(texts) + 1, np.int64)
    offs[1:] = np.cumsum([len(t) for t in texts])
    s2 = ctx.score_text(Extractor.make(), arena, offs, w, 0.25)
    so = oracle.score_batch(OEx.make(), arena, offs, w, 0.25)
    assert (s.view(np.uint64) == s2.view(np.uint64)).all()
    assert (s.view(np.uint64) == so.view(np.uint64)).all()


@pytest.mark.parametrize("n", [4097, 5000, 65536, 100_003, 1 << 20])
def test_priority_order_radix_sizes(ctx, n):
    """The onesweep radix path from just above the bitonic switch to 2^20
    keys (one to 147 tiles of look-back): ties in score and tie rank, +-0.0,
    boosts, against numpy's lexsort of the same keys."""
    rng = np.random.default_rng(n)
    score = rng.choice(np.concatenate([rng.normal(size=300), [0.0, -0.0]]), size=n)
    tie = rng.integers(0, 50, size=n).astype(np.uint32)
    boosted = (rng.random(n) < 0.05).astype(np.uint8)
    got = ctx.priority_order(score, tie, boosted)
    # select_batch's order: boosted first, then (score, tie), then index; -0.0 == +0.0
    s = np.where(score == 0, 0.0, score)
    # boosted keys compare by (tie, index) only
    want = np.lexsort((np.arange(n), tie, np.where(boosted == 1, 0.0, s), 1 - boosted.astype(np.int64)))
    assert (got == want).all()


@pytest.mark.parametrize("run", [1, 2, 31, 32, 33, 200])
@pytest.mark.parametrize("ties", [True, False])
def test_priority_order_high_word_runs(ctx, run, ties):
    """The speculative high-word sort (sort.cu radix_fixup): keys whose top
    32 bits repeat in shuffled runs of `run` keys with distinct or equal low
    words, a few boosted keys (one run of top word 0), tie ranks that order
    equal scores. Runs up to kFixRun = 32 are placed by the fixup, longer
    ones make the full LSD passes run; both against numpy's lexsort."""
    n = 150_000
    rng = np.random.default_rng(100 + run)
    nb = n // run + 1
    top = (rng.normal(size=nb) * 10).view(np.uint64) & np.uint64(0xFFFFFFFF00000000)
    low = rng.integers(0, 2**32, size=(nb, run), dtype=np.uint64)
    low[:, 0] = low[:, -1]  # equal full scores inside a run
    score = (top[:, None] | low).reshape(-1)[:n].view(np.float64)[rng.permutation(n)]
    tie = rng.integers(0, 3, size=n) if ties else np.zeros(n)  # all-zero ranks: no tie passes
    tie = tie.astype(np.uint32)
    boosted = (rng.random(n) < 1e-4).astype(np.uint8)
    got = ctx.priority_order(score, tie, boosted)
    want = np.lexsort((np.arange(n), tie, np.where(boosted == 1, 0.0, score), 1 - boosted.astype(np.int64)))
    assert (got == want).all()



def test_c4_hard_variant_scores_bit_identical(ctx, oracle):
    """SURVEY 8(d)'s hard C4 variant (prompts padded to 512 tokens with random
    6-letter words: ~3.4 KB, ~1,520 touched buckets per prompt, every list
    longer than the old 512-entry ring slot): exact scores bit-identical to
    the oracle, fast scores within the fp32 tolerance."""
    from paper_2510_03243_b200 import MODE_FAST, Extractor, Workload
    wl = Workload.synthesize(3000, 31, pad_tokens=512, pad_seed=5, pad_words="random6")
    w = np.random.default_rng(9).normal(size=4096) * 0.05
    got = ctx.score_text(Extractor.make(), wl.text, wl.offsets, w, 0.0)
    want = oracle.score_batch(OEx.make(), wl.text, wl.offsets, w, 0.0, threads=os.cpu_count())
    assert (got.view(np.uint64) == want.view(np.uint64)).all()
    fast = ctx.score_text(Extractor.make(), wl.text, wl.offsets, w, 0.0, mode=MODE_FAST)
    assert np.abs(fast - want).max() < 1e-5 * np.abs(w).sum()


def test_fused_ring_many_tiny_and_mixed_prompts(ctx, oracle):
    """The fused kernel's ring hand-off under stress: 200,000 prompts that are
    mostly empty or one token (hashing warps finish prompts far faster than
    the chain warps consume rounds, so slots wrap many times), mixed with a
    few ~1,700-bucket prompts (lists past the old 512-entry slot) and a few
    too long for a slot (the hashing warp's own chain): every exact score
    bit-identical to the oracle."""
    from paper_2510_03243_b200 import Extractor, pack_texts
    rng = np.random.default_rng(77)
    words = [bytes(rng.integers(97, 123, size=rng.integers(1, 9)).astype(np.uint8)) for _ in range(5000)]
    texts = []
    for k in range(200_000):
        r = rng.random()
        if r < 0.3:
            texts.append(b"")
        elif r < 0.9:
            texts.append(words[rng.integers(0, len(words))])
        elif r < 0.999:
            texts.append(b" ".join(words[j] for j in rng.integers(0, len(words), size=rng.integers(2, 60))))
        elif r < 0.9995:
            texts.append(b" ".join(bytes(rng.integers(97, 123, size=6).astype(np.uint8)) for _ in range(500)))
        else:
            texts.append(b" ".join(bytes(rng.integers(97, 123, size=6).astype(np.uint8)) for _ in range(1400)))
    arena, offs = pack_texts(texts)
    w = np.random.default_rng(5).normal(size=4096)
    got = ctx.score_text(Extractor.make(), arena, offs, w, 0.5)
    want = oracle.score_batch(OEx.make(), arena, offs, w, 0.5, threads=os.cpu_count())
    assert (got.view(np.uint64) == want.view(np.uint64)).all()
