"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
library itself (oracle/_ref/libpars_ref.so, compiled from
/root/reference/proj/src by `make -C oracle ref`).

Run here (the build container, where /root/reference exists):
    python tests/golden/make_golden.py
The fixtures are committed; the GPU box never needs /root/reference.
Doubles are stored as C99 hex-float strings so they round-trip bit-exactly.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.bind import Extractor, Ref, fnv64_array  # noqa: E402

OUT = Path(__file__).resolve().parent


def hx(a):
    return [float(x).hex() for x in np.asarray(a, np.float64).ravel()]


def ex_desc(e: Extractor):
    return dict(kind=int(e.kind), dim=int(e.dim), norm=int(e.norm),
                word=[int(e.word[i]) for i in range(e.n_word)],
                char=[int(e.chr[i]) for i in range(e.n_char)])


EXTRACTORS = [
    Extractor.make(),
    Extractor.make(norm="none"),
    Extractor.make(dim=8),
    Extractor.make(dim=12, word=(1, 2), char=(2, 4)),
    Extractor.make(dim=3, norm="none"),
    Extractor.make(dim=1000, word=(2,), char=()),
    Extractor.make(dim=4096, word=(), char=(3,), norm="none"),
    Extractor.make(dim=65536, word=(1, 3), char=(1, 5)),
    Extractor.make(dim=1, word=(1,), char=(3,)),
    Extractor.make(dim=97, word=(1, 2, 3), char=(3,)),
]

TEXTS = [
    b"", b"   ", b"x", b"a b c", b"ab cd", b"abcd", b"tok tok", b"alpha beta", b"alpha gamma",
    b"the quick brown fox a1", b"len80 lvl0 lvl1 w3 w4", b"some words here",
    b"\t\n\v\f\r mixed\twhite\nspace\vtokens\fhere\r", b"\x80\xff\xfe high-bit \xc3\xa9t\xc3\xa9",
    b"  leading and trailing  ", b"a" * 300, b"ab " * 200, b"x" * 5000 + b" y",
    b"w1 w2 w3 w4 w5 w6 w7 w8 w9 w10 w11 w12 w13 w14 w15 w16 w17 w18 w19 w20 w21 w22 w23 w24 "
    b"w25 w26 w27 w28 w29 w30 w31 w32 w33 w34 w35 w36",
    b"\x00nul\x00inside", b"a\x1fb", b"lvl" * 40,
]


def gen_features(R: Ref):
    cases = []
    ds = R.synthesize(40, 9)
    texts = TEXTS + [ds.prompt(i) for i in range(ds.n)]
    for e in EXTRACTORS:
        for t in texts:
            idx, val = R.extract(e, t)
            cases.append(dict(extractor=ex_desc(e), text=t.hex(), idx=idx.tolist(), val=hx(val)))
    emb_cases = []
    e = Extractor.make(dim=5, kind="embedding", norm="l2")
    rng = np.random.default_rng(3)
    for k in range(6):
        x = rng.normal(size=5)
        if k == 0:
            x[:] = 0.0
        if k == 1:
            x[2] = 0.0
        idx, val = R.extract(e, b"ignored", emb=x)
        emb_cases.append(dict(x=hx(x), idx=idx.tolist(), val=hx(val)))
    (OUT / "features.json").write_text(json.dumps(dict(cases=cases, embedding=emb_cases)))
    print("features.json:", len(cases), "cases")


def gen_models(R: Ref):
    ex = Extractor.make()
    full = R.synthesize(4000, 21)
    tr, va = R.split(full, 0.2, 21)
    w, bias, lt = R.train(tr, ex, seed=21)
    tau, counts = R.evaluate_ranking(ex, va, w, bias)
    wl = R.synthesize(500, 22)
    s500 = R.score_batch(ex, wl, w, bias)
    ids = wl.ids()
    order500 = R.select_batch(np.zeros(wl.n), ids, s500, np.zeros(wl.n, np.uint8), 0.0, wl.n)
    # C1: first 1,024 records with prompt_len <= 128 of gen(2048, seed 22)
    g = R.synthesize(2048, 22)
    sel = np.nonzero(g.prompt_len <= 128)[0][:1024]
    c1 = R.subset(g, sel)
    s1 = R.score_batch(ex, c1, w, bias)
    ids1 = c1.ids()
    order1 = R.select_batch(np.zeros(c1.n), ids1, s1, np.zeros(c1.n, np.uint8), 0.0, c1.n)
    # C2: one epoch on gen(8192, seed 21)
    d2 = R.synthesize(8192, 21)
    w2, b2, lt2 = R.train(d2, ex, seed=21, epochs=1)
    np.savez_compressed(OUT / "readme_model.npz", weights=w, loss_trace=lt, s500=s500,
                        order500=order500, c1_index=sel, c1_scores=s1, c1_order=order1,
                        c2_weights=w2, c2_loss=lt2)
    meta = dict(
        readme=dict(loss_trace=hx(lt), weights_fnv=fnv64_array(w), bias=float(bias).hex(),
                    val_tau=float(tau).hex(), val_counts=[int(c) for c in counts]),
        workload500=dict(scores_head=hx(s500[:3]), order_head=order500[:5].tolist(),
                         order_fnv=fnv64_array(order500.astype(np.uint64))),
        c1=dict(n=int(c1.n), last_id=ids1[-1], scores_fnv=fnv64_array(s1),
                order_head=order1[:5].tolist(), order_fnv=fnv64_array(order1.astype(np.uint64))),
        c2=dict(loss0=float(lt2[0]).hex(), weights_fnv=fnv64_array(w2)),
    )
    (OUT / "models.json").write_text(json.dumps(meta, indent=1))
    print(json.dumps(meta, indent=1))


def gen_train_small(R: Ref):
    cases = []
    for (n, seed, epochs, ppe, batch, lr, margin, delta, dim) in [
        (300, 4, 3, 2000, 128, 0.1, 1.0, 0.2, 4096),
        (120, 7, 2, 777, 50, 0.5, 0.5, 0.0, 256),
        (200, 11, 2, 1500, 1, 0.05, 2.0, 0.5, 4096),
        (64, 3, 1, 3000, 1000, 0.2, 1.0, 0.3, 64),
    ]:
        ds = R.synthesize(n, seed)
        ex = Extractor.make(dim=dim)
        w, b, lt = R.train(ds, ex, seed=seed, epochs=epochs, ppe=ppe, batch=batch, lr=lr,
                           margin=margin, delta=delta)
        cases.append(dict(n=n, seed=seed, epochs=epochs, ppe=ppe, batch=batch, lr=lr,
                          margin=margin, delta=delta, dim=dim, loss_trace=hx(lt),
                          weights_fnv=fnv64_array(w), weights=hx(w) if dim <= 256 else None))
    (OUT / "train_small.json").write_text(json.dumps(cases))
    print("train_small.json:", len(cases))


def gen_pairs(R: Ref):
    cases = []
    for (n, seed, delta, maxp, pseed) in [(200, 1, 0.2, 500, 7), (200, 1, 0.0, 300, 8),
                                          (50, 2, 0.5, 1000, 9), (1000, 3, 0.9, 400, 10)]:
        ds = R.synthesize(n, seed)
        a, b, y, rel = R.build_pairs(ds, delta, maxp, pseed)
        cases.append(dict(lengths=ds.output_len.tolist(), delta=delta, max_pairs=maxp,
                          seed=pseed, a=a.tolist(), b=b.tolist(), y=y.tolist(), rel=hx(rel)))
    (OUT / "pairs.json").write_text(json.dumps(cases))
    print("pairs.json:", len(cases))


def gen_select(R: Ref):
    rng = np.random.default_rng(11)
    cases = []
    for k in range(30):
        n = int(rng.integers(1, 60))
        arrival = rng.choice([0.0, 0.5, 1.0, 1.5], size=n)
        ids = [f"r{int(rng.integers(0, 8))}" for _ in range(n)]
        score = rng.choice([-1.0, 0.0, -0.0, 0.25, 2.0, rng.normal()], size=n)
        boosted = (rng.random(n) < 0.2).astype(np.uint8)
        now = 2.0
        order = R.select_batch(arrival, ids, score, boosted, now, n)
        cases.append(dict(arrival=hx(arrival), ids=ids, score=hx(score),
                          boosted=boosted.tolist(), now=now, order=order.tolist()))
    (OUT / "select.json").write_text(json.dumps(cases))
    print("select.json:", len(cases))


def gen_tau(R: Ref):
    rng = np.random.default_rng(5)
    cases = []
    for n in [2, 3, 10, 100, 777]:
        x = rng.integers(0, 7, size=n).astype(np.float64)
        y = rng.normal(size=n).round(1)
        tau, counts = R.kendall(x, y)
        cases.append(dict(x=hx(x), y=hx(y), tau=float(tau).hex(), counts=[int(c) for c in counts]))
    (OUT / "tau.json").write_text(json.dumps(cases))
    print("tau.json:", len(cases))


def mask_count(lens: np.ndarray, delta: float) -> int:
    """Exhaustive Eq. 1 count over unordered pairs with the reference's
    formula (pairs.hpp:21-24; IEEE double division, identical to C)."""
    lens = lens.astype(np.int64)
    n = len(lens)
    total = 0
    B = 2048
    for i0 in range(0, n, B):
        a = lens[i0:i0 + B][:, None]
        j0 = i0
        b = lens[j0:][None, :]
        d = np.abs(a - b).astype(np.float64)
        m = np.maximum(a, b).astype(np.float64)
        keep = (a != b) & ~((d / m) < delta)
        ii = np.arange(i0, i0 + a.shape[0])[:, None]
        jj = np.arange(j0, n)[None, :]
        total += int(np.count_nonzero(keep & (jj > ii)))
    return total


def gen_mask_counts(R: Ref):
    out = {}
    for (n, seed, mu, sigma) in [(8192, 21, 5.0, 1.2), (1024, 22, 4.0, 1.0), (65536, 25, 5.0, 1.2)]:
        ds = R.synthesize(n, seed, mu=mu, sigma=sigma)
        out[f"{n}_{seed}"] = dict(n=n, seed=seed, mu=mu, sigma=sigma, delta=0.2,
                                  kept=mask_count(ds.output_len, 0.2))
        print(out[f"{n}_{seed}"])
    (OUT / "mask_counts.json").write_text(json.dumps(out, indent=1))


def gen_synth(R: Ref):
    """Hashes of the reference generator's output (dataset.cpp:204-297)."""
    out = []
    for (n, seed) in [(500, 22), (4000, 21), (2048, 22), (8192, 21)]:
        ds = R.synthesize(n, seed)
        out.append(dict(n=n, seed=seed, text_fnv=fnv64_array(np.frombuffer(
            ds.text.tobytes() + b"\0" * ((-len(ds.text)) % 8), np.uint64)),
            offsets_fnv=fnv64_array(ds.offs.astype(np.uint64)),
            output_len_fnv=fnv64_array(ds.output_len.astype(np.uint64)),
            prompt_len_fnv=fnv64_array(ds.prompt_len.astype(np.uint64))))
    (OUT / "synth.json").write_text(json.dumps(out, indent=1))
    print("synth.json", len(out))


def gen_sim(R: Ref):
    """README burst-500 comparison (proj/README.md:26-36), in-library."""
    ex = Extractor.make()
    full = R.synthesize(4000, 21)
    tr, _ = R.split(full, 0.2, 21)
    w, bias, _ = R.train(tr, ex, seed=21)
    wl = R.synthesize(500, 22)
    res = {}
    for pol in ("fcfs", "oracle", "pars"):
        r = R.simulate(wl, None, pol, ex=ex, w=w, bias=bias)
        res[pol] = dict(mean_ms=float(r["mean_ms"]).hex(), p90_ms=float(r["p90_ms"]).hex(),
                        iterations=int(r["iterations"]), seconds=float(r["seconds"]).hex(),
                        completion=r["record"].tolist(), finish=hx(r["finish"]))
    (OUT / "sim_burst500.json").write_text(json.dumps(res))
    print({k: (float.fromhex(v["mean_ms"]), v["iterations"]) for k, v in res.items()})


if __name__ == "__main__":
    R = Ref()
    R.set_threads(1)
    which = sys.argv[1:] or ["features", "models", "train_small", "pairs", "select", "tau",
                             "synth", "sim", "mask_counts"]
    for w in which:
        globals()[f"gen_{w}"](R)
