"""CPU tests of the C ABI library: it loads, exports every symbol
include/pars_cuda.h declares, and its host-side functions (build_pairs, the
Eq. 1 table, tie ranks, the workload generator) match the reference. No
device compute here."""
import ctypes as C
import re

import numpy as np
import pytest

from conftest import ROOT, golden, unhex


def header_symbols():
    txt = (ROOT / "include" / "pars_cuda.h").read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pars_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2510_03243_b200 import lib
    L = lib()
    syms = header_symbols()
    assert len(syms) >= 35
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_version_and_no_device_is_an_error_not_a_fallback():
    from paper_2510_03243_b200 import Context, ParsError, device_count, lib
    assert b"sm_100a" in lib().pars_version()
    if device_count() == 0:
        with pytest.raises(ParsError):
            Context(0)


def test_build_pairs_matches_reference_goldens():
    from paper_2510_03243_b200 import build_pairs
    for c in golden("pairs.json"):
        a, b, y, rel = build_pairs(np.array(c["lengths"]), c["delta"], c["max_pairs"], c["seed"])
        assert a.tolist() == c["a"] and b.tolist() == c["b"] and y.tolist() == c["y"]
        assert [float(r).hex() for r in rel] == c["rel"]


def test_build_pairs_errors_use_reference_messages():
    from paper_2510_03243_b200 import ParsError, build_pairs
    with pytest.raises(ParsError, match="no informative pairs"):
        build_pairs(np.full(10, 7), 0.2, 10, 1)
    with pytest.raises(ParsError, match=r"build_pairs: delta 1 outside \[0, 1\)"):
        build_pairs(np.arange(1, 10), 1.0, 10, 1)
    with pytest.raises(ParsError, match="max_pairs must be >= 1"):
        build_pairs(np.arange(1, 10), 0.2, 0, 1)


def test_build_pairs_matches_reference_live(ref):
    from paper_2510_03243_b200 import build_pairs
    ds = ref.synthesize(3000, 17)
    for delta, seed in [(0.2, 1), (0.0, 2), (0.6, 3)]:
        a, b, y, rel = build_pairs(ds.output_len, delta, 5000, seed)
        ra, rb, ry, rrel = ref.build_pairs(ds, delta, 5000, seed)
        assert (a == ra).all() and (b == rb).all() and (y == ry).all() and (rel == rrel).all()


def test_length_gap_table_matches_oracle(oracle):
    from paper_2510_03243_b200 import length_gap_table
    for delta in (0.0, 0.05, 0.2, 1 / 3, 0.5, 0.75, 0.999):
        assert (length_gap_table(delta, 5000) == oracle.dmin_table(delta, 5000)).all()


def test_tie_ranks_order_by_arrival_then_id_bytes():
    from paper_2510_03243_b200 import tie_ranks
    arrival = np.array([1.0, 0.0, 1.0, 0.0, 1.0, 0.5])
    ids = ["b", "z", "a", "z", "b\xff", "m"]
    r = tie_ranks(arrival, ids)
    # (0,z) (0,z) tie -> rank 0; (0.5,m) 1; (1,a) 2; (1,b) 3; (1,b\xff) 4
    assert r.tolist() == [3, 0, 2, 0, 4, 1]


def test_workload_generator_is_bit_identical_to_reference():
    from oracle.bind import fnv64_array
    from paper_2510_03243_b200 import Workload
    for c in golden("synth.json"):
        w = Workload.synthesize(c["n"], c["seed"])
        t = w.text.tobytes()
        t += b"\0" * ((-len(t)) % 8)
        assert fnv64_array(np.frombuffer(t, np.uint64)) == c["text_fnv"]
        assert fnv64_array(w.offsets.astype(np.uint64)) == c["offsets_fnv"]
        assert fnv64_array(w.output_len.astype(np.uint64)) == c["output_len_fnv"]
        assert fnv64_array(w.prompt_len.astype(np.uint64)) == c["prompt_len_fnv"]
        w.close()


def test_workload_padding_to_fixed_token_count():
    from paper_2510_03243_b200 import Workload
    w = Workload.synthesize(50, 31, pad_tokens=512, pad_seed=5)
    for i in range(len(w)):
        toks = w.prompt(i).split()
        assert len(toks) == 512 == w.prompt_len[i]
    w.close()


def test_baseline_samplers_match_reference(ref):
    """pars_pointwise_order / pars_listmle_lists (host, the epoch order and
    lists of train()'s PointwiseL1 / ListMLE objectives) against the same
    samplers over the reference's Rng (oracle/ref_capi.cpp)."""
    from paper_2510_03243_b200 import lib
    for n, seed in ((1, 3), (2, 9), (1000, 0x1234), (4097, 2**63 + 5)):
        got = np.zeros(n, np.uint32)
        assert lib().pars_pointwise_order(n, C.c_uint64(seed), got.ctypes.data) == 0
        assert got.tolist() == ref.pointwise_order(n, seed).tolist()
    for n, nlists, k, seed in ((600, 50, 10, 7), (5, 11, 10, 8), (300, 20, 2, 2**40)):
        ds = ref.synthesize(n, 40 + n)
        ids = ds.ids()
        bs = [i.encode() for i in ids]
        offs = np.zeros(n + 1, np.int64)
        offs[1:] = np.cumsum([len(b) for b in bs])
        arena = np.frombuffer(b"".join(bs) + b"\0", np.uint8)
        kk = min(k, n)
        got = np.zeros(nlists * kk, np.uint32)
        lens = np.ascontiguousarray(ds.output_len, np.int64)
        assert lib().pars_listmle_lists(lens.ctypes.data, arena.ctypes.data, offs.ctypes.data, n,
                                        nlists, k, C.c_uint64(seed), got.ctypes.data) == 0
        assert got.tolist() == ref.listmle_lists(ds, nlists, k, seed).tolist()


def test_tie_ranks_sorted_fast_path_equals_general_path():
    """Inputs already in (arrival, id) order take a linear pass; a shuffle of
    the same requests takes the sort. Every request must get the same dense
    rank either way (equal keys share one)."""
    from paper_2510_03243_b200 import tie_ranks
    rng = np.random.default_rng(11)
    n = 5000
    arrival = np.sort(np.round(rng.random(n) * 50, 1))
    ids = ["p%04d" % rng.integers(0, 3000) for _ in range(n)]
    key = sorted(range(n), key=lambda i: (arrival[i], ids[i].encode()))
    arrival, ids = arrival[key], [ids[i] for i in key]
    r_sorted = tie_ranks(arrival, ids)
    perm = rng.permutation(n)
    r_perm = tie_ranks(arrival[perm], [ids[i] for i in perm])
    assert (r_perm == r_sorted[perm]).all()
    assert r_sorted[0] == 0 and (np.diff(r_sorted.astype(np.int64)) >= 0).all()
    assert r_sorted[-1] + 1 == len({(a, i) for a, i in zip(arrival, ids)})
