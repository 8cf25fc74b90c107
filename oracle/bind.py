"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the checker libraries.

* ``Oracle``  -> oracle/liboracle.so, the plain-C restatement (pars_oracle.c).
* ``Ref``     -> oracle/_ref/libpars_ref.so, the unmodified reference library
  compiled from /root/reference/proj/src by oracle/Makefile (present in the
  build container and shipped prebuilt to the GPU box; never rebuilt there).

Only tests/, tests/golden/make_golden.py, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libpars_ref.so"


class Extractor(C.Structure):
    """pars::FeatureExtractor (features.hpp:17-25) as a C POD."""

    _fields_ = [
        ("kind", C.c_int32),
        ("dim", C.c_uint32),
        ("norm", C.c_int32),
        ("n_word", C.c_int32),
        ("n_char", C.c_int32),
        ("word", C.c_int32 * 8),
        ("chr", C.c_int32 * 8),
    ]

    @classmethod
    def make(cls, dim=4096, word=(1,), char=(3,), norm="l2", kind="hashed"):
        e = cls()
        e.kind = 0 if kind == "hashed" else 1
        e.dim = dim
        e.norm = 1 if norm == "l2" else 0
        e.n_word = len(word)
        e.n_char = len(char)
        for i, w in enumerate(word):
            e.word[i] = w
        for i, c in enumerate(char):
            e.chr[i] = c
        return e


P = np.ctypeslib.ndpointer
_f64 = P(np.float64, flags="C_CONTIGUOUS")
_i64 = P(np.int64, flags="C_CONTIGUOUS")
_u64 = P(np.uint64, flags="C_CONTIGUOUS")
_u32 = P(np.uint32, flags="C_CONTIGUOUS")
_i32 = P(np.int32, flags="C_CONTIGUOUS")
_u8 = P(np.uint8, flags="C_CONTIGUOUS")


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class OracleError(RuntimeError):
    pass


class Oracle:
    """Plain-C restatement of the reference hot path (pars_oracle.c)."""

    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        L = self.L = C.CDLL(str(path))
        L.po_last_error.restype = C.c_char_p
        L.po_extract.restype = C.c_int64
        L.po_extract_all.restype = C.c_int64
        L.po_build_pairs.restype = C.c_int64
        L.po_rel_diff.restype = C.c_double
        L.po_rel_diff.argtypes = [C.c_int64, C.c_int64]
        L.po_margin_loss.restype = C.c_double
        L.po_margin_loss.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double]
        L.po_splitmix64.restype = C.c_uint64
        L.po_splitmix64.argtypes = [C.c_uint64]
        L.po_derive_seed.restype = C.c_uint64
        L.po_derive_seed.argtypes = [C.c_uint64, C.c_uint64]

    def _err(self):
        return OracleError(self.L.po_last_error().decode())

    def extract(self, ex: Extractor, text: bytes, emb=None):
        cap = max(1, len(text) * 16 + ex.dim)
        idx = np.zeros(cap, np.uint32)
        val = np.zeros(cap, np.float64)
        embc = None if emb is None else np.ascontiguousarray(emb, np.float64)
        n = self.L.po_extract(C.byref(ex), C.c_char_p(text), C.c_int64(len(text)),
                              _ptr(embc), C.c_int64(0 if emb is None else len(emb)),
                              _ptr(idx), _ptr(val), C.c_int64(cap))
        if n < 0:
            raise self._err()
        return idx[:n].copy(), val[:n].copy()

    def extract_all(self, ex, text: np.ndarray, offs: np.ndarray):
        n = len(offs) - 1
        rp = np.zeros(n + 1, np.int64)
        cap = int(offs[-1]) * (ex.n_char or 1) + n * 4 + 16
        cap = cap * max(1, ex.n_word + ex.n_char)
        idx = np.zeros(cap, np.uint32)
        val = np.zeros(cap, np.float64)
        tot = self.L.po_extract_all(C.byref(ex), _ptr(text), _ptr(offs), C.c_int64(n),
                                    _ptr(rp), _ptr(idx), _ptr(val), C.c_int64(cap))
        if tot < 0:
            raise self._err()
        return rp, idx[:tot].copy(), val[:tot].copy()

    def score_batch(self, ex, text, offs, w, bias=0.0, threads=1):
        n = len(offs) - 1
        out = np.zeros(n, np.float64)
        rc = self.L.po_score_batch(C.byref(ex), _ptr(text), _ptr(offs), C.c_int64(n),
                                   _ptr(np.ascontiguousarray(w, np.float64)),
                                   C.c_double(bias), _ptr(out), C.c_int(threads))
        if rc != 0:
            raise self._err()
        return out

    def score_dense(self, ex, X, w, bias=0.0):
        X = np.ascontiguousarray(X, np.float64)
        out = np.zeros(X.shape[0], np.float64)
        rc = self.L.po_score_dense(C.byref(ex), _ptr(X), C.c_int64(X.shape[0]),
                                   _ptr(np.ascontiguousarray(w, np.float64)),
                                   C.c_double(bias), _ptr(out))
        if rc != 0:
            raise self._err()
        return out

    def rel_diff(self, a, b):
        return self.L.po_rel_diff(a, b)

    def margin_loss(self, sa, sb, y, m):
        return self.L.po_margin_loss(sa, sb, y, m)

    def dmin_table(self, delta, max_len):
        t = np.zeros(max_len + 1, np.int32)
        self.L.po_dmin_table(C.c_double(delta), C.c_int64(max_len), _ptr(t))
        return t

    def build_pairs(self, lens, delta, max_pairs, seed):
        lens = np.ascontiguousarray(lens, np.int64)
        a = np.zeros(max_pairs, np.uint32)
        b = np.zeros(max_pairs, np.uint32)
        y = np.zeros(max_pairs, np.int32)
        rel = np.zeros(max_pairs, np.float64)
        n = self.L.po_build_pairs(_ptr(lens), C.c_int64(len(lens)), C.c_double(delta),
                                  C.c_uint64(max_pairs), C.c_uint64(seed),
                                  _ptr(a), _ptr(b), _ptr(y), _ptr(rel))
        if n < 0:
            raise self._err()
        return a[:n].copy(), b[:n].copy(), y[:n].copy(), rel[:n].copy()

    def derive_seed(self, seed, stream):
        return self.L.po_derive_seed(seed, stream)

    def sgd_epoch(self, rp, idx, val, dim, a, b, y, batch, lr, margin, w, bias=0.0):
        w = np.array(w, np.float64)
        el = C.c_double(0.0)
        act = C.c_uint64(0)
        self.L.po_sgd_epoch(_ptr(rp), _ptr(idx), _ptr(val), C.c_uint32(dim),
                            _ptr(np.ascontiguousarray(a, np.uint32)),
                            _ptr(np.ascontiguousarray(b, np.uint32)),
                            _ptr(np.ascontiguousarray(y, np.int32)),
                            C.c_int64(len(a)), C.c_int(batch), C.c_double(lr),
                            C.c_double(margin), _ptr(w), C.c_double(bias),
                            C.byref(el), C.byref(act))
        return w, el.value, act.value

    def train_pairwise(self, rp, idx, val, lens, dim, delta=0.2, margin=1.0, epochs=5,
                       batch=128, lr=0.1, seed=0, ppe=100000):
        w = np.zeros(dim, np.float64)
        bias = C.c_double(0.0)
        lt = np.zeros(max(epochs, 1), np.float64)
        lens = np.ascontiguousarray(lens, np.int64)
        rc = self.L.po_train_pairwise(_ptr(rp), _ptr(idx), _ptr(val), _ptr(lens),
                                      C.c_int64(len(lens)), C.c_uint32(dim), C.c_double(delta),
                                      C.c_double(margin), C.c_int(epochs), C.c_int(batch),
                                      C.c_double(lr), C.c_uint64(seed), C.c_uint64(ppe),
                                      _ptr(w), C.byref(bias), _ptr(lt))
        if rc != 0:
            raise self._err()
        return w, bias.value, lt[:epochs].copy()

    def allpairs(self, s, lens, delta, margin, threads=1):
        s = np.ascontiguousarray(s, np.float64)
        lens = np.ascontiguousarray(lens, np.int64)
        c = np.zeros(len(s), np.int32)
        kept, act, loss = C.c_uint64(), C.c_uint64(), C.c_double()
        self.L.po_allpairs(_ptr(s), _ptr(lens), C.c_int64(len(s)), C.c_double(delta),
                           C.c_double(margin), _ptr(c), C.byref(kept), C.byref(act),
                           C.byref(loss), C.c_int(threads))
        return c, kept.value, act.value, loss.value

    def xt_c(self, rp, idx, val, coeff, dim):
        g = np.zeros(dim, np.float64)
        self.L.po_xt_c(_ptr(rp), _ptr(idx), _ptr(val), C.c_int64(len(rp) - 1),
                       _ptr(np.ascontiguousarray(coeff, np.int32)), C.c_uint32(dim), _ptr(g))
        return g

    def select_order(self, arrival, ids, score, boosted, now):
        n = len(arrival)
        arena, offs = ids_arena(ids)
        order = np.zeros(n, np.int64)
        rc = self.L.po_select_order(C.c_int64(n), _ptr(np.ascontiguousarray(arrival, np.float64)),
                                    C.c_char_p(arena), _ptr(offs),
                                    _ptr(np.ascontiguousarray(score, np.float64)),
                                    _ptr(np.ascontiguousarray(boosted, np.uint8)),
                                    C.c_double(now), _ptr(order))
        if rc != 0:
            raise self._err()
        return order

    def kendall(self, x, y, threads=1):
        counts = np.zeros(5, np.uint64)
        tau = C.c_double()
        rc = self.L.po_kendall(_ptr(np.ascontiguousarray(x, np.float64)),
                               _ptr(np.ascontiguousarray(y, np.float64)),
                               C.c_int64(len(x)), _ptr(counts), C.byref(tau), C.c_int(threads))
        if rc != 0:
            raise self._err()
        return tau.value, counts


def ids_arena(ids):
    bs = [i.encode() if isinstance(i, str) else bytes(i) for i in ids]
    offs = np.zeros(len(bs) + 1, np.int64)
    offs[1:] = np.cumsum([len(b) for b in bs])
    return b"".join(bs) + b"\0", offs


class Dataset:
    """Flat view of a pars::Dataset living inside libpars_ref.so."""

    def __init__(self, ref: "Ref", handle, export=True):
        if not handle:
            raise OracleError(ref.L.ref_last_error().decode("utf-8", "replace"))
        self.ref, self.h = ref, handle
        L = ref.L
        n = L.ref_dataset_size(handle)
        self.n = n
        if not export:  # handle only (no flat copy of the records)
            return
        nb = L.ref_dataset_text_bytes(handle)
        ed = L.ref_dataset_embed_dim(handle)
        self.text = np.zeros(max(nb, 1), np.uint8)
        self.offs = np.zeros(n + 1, np.int64)
        self.output_len = np.zeros(n, np.int64)
        self.prompt_len = np.zeros(n, np.int64)
        self.embedding = np.zeros((n, ed), np.float64) if ed > 0 else None
        L.ref_dataset_export(handle, _ptr(self.text), _ptr(self.offs), _ptr(self.output_len),
                             _ptr(self.prompt_len), _ptr(self.embedding))
        self.n = n

    def __len__(self):
        return self.n

    def prompt(self, i) -> bytes:
        return self.text[self.offs[i]:self.offs[i + 1]].tobytes()

    def ids(self):
        buf = C.create_string_buffer(64)
        out = []
        for i in range(self.n):
            self.ref.L.ref_dataset_id(self.h, C.c_uint64(i), buf, C.c_int64(64))
            out.append(buf.value.decode())
        return out

    def __del__(self):
        try:
            self.ref.L.ref_dataset_free(self.h)
        except Exception:
            pass


class Ref:
    """The unmodified reference library (oracle/_ref/libpars_ref.so)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run `make -C oracle ref`)")
        L = self.L = C.CDLL(str(path))
        L.ref_last_error.restype = C.c_char_p
        for name in ("ref_synthesize", "ref_dataset_from_arrays", "ref_split", "ref_subset",
                     "ref_simulate", "ref_load_dataset"):
            getattr(L, name).restype = C.c_void_p
        L.ref_load_dataset.argtypes = [C.c_char_p, C.c_int64]
        L.ref_save_dataset.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_dataset_samples.restype = C.c_int64
        L.ref_dataset_samples.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_int64]
        L.ref_synthesize.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_uint64,
                                     C.c_int64, C.c_int64]
        L.ref_split.argtypes = [C.c_void_p, C.c_double, C.c_uint64, C.c_int]
        L.ref_subset.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.ref_dataset_from_arrays.argtypes = [C.c_void_p] * 4 + [C.c_int64, C.c_void_p, C.c_int64]
        for name in ("ref_dataset_size", "ref_sim_iterations", "ref_sim_count"):
            getattr(L, name).restype = C.c_uint64
            getattr(L, name).argtypes = [C.c_void_p]
        for name in ("ref_dataset_text_bytes", "ref_dataset_embed_dim"):
            getattr(L, name).restype = C.c_int64
            getattr(L, name).argtypes = [C.c_void_p]
        L.ref_dataset_export.argtypes = [C.c_void_p] * 6
        L.ref_dataset_id.argtypes = [C.c_void_p, C.c_uint64, C.c_char_p, C.c_int64]
        L.ref_dataset_free.argtypes = [C.c_void_p]
        L.ref_sim_free.argtypes = [C.c_void_p]
        L.ref_sim_seconds.restype = C.c_double
        L.ref_sim_seconds.argtypes = [C.c_void_p]
        L.ref_sim_requests.argtypes = [C.c_void_p] * 7
        L.ref_sim_summary.argtypes = [C.c_void_p] * 3
        L.ref_simulate.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                   C.c_double, C.c_int, C.c_double, C.c_int]
        L.ref_extract.restype = C.c_int64
        L.ref_extract_all.restype = C.c_int64
        L.ref_extract_all.argtypes = [C.c_void_p] * 5 + [C.c_int64]
        L.ref_build_pairs.restype = C.c_int64
        L.ref_build_pairs.argtypes = [C.c_void_p, C.c_double, C.c_uint64, C.c_uint64] + [C.c_void_p] * 4
        L.ref_select_batch.restype = C.c_int64
        L.ref_relative_length_difference.restype = C.c_double
        L.ref_relative_length_difference.argtypes = [C.c_int64, C.c_int64]
        L.ref_margin_ranking_loss.restype = C.c_double
        L.ref_margin_ranking_loss.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double]
        L.ref_score_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p]
        L.ref_evaluate_ranking.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                           C.c_void_p, C.c_void_p]
        L.ref_train.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int,
                                C.c_int, C.c_double, C.c_uint64, C.c_uint64, C.c_uint64,
                                C.c_int, C.c_void_p,
                                C.c_void_p, C.c_void_p]
        L.ref_pointwise_order.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p]
        L.ref_listmle_lists.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.c_void_p]
        L.ref_poisson.argtypes = [C.c_void_p, C.c_double, C.c_uint64, C.c_void_p]
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_pad_dataset.argtypes = [C.c_void_p, C.c_int64, C.c_uint64]
        L.ref_score_order.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                      C.c_void_p]

    def _err(self):
        return OracleError(self.L.ref_last_error().decode("utf-8", "replace"))

    def set_threads(self, n):
        self.L.ref_set_threads(n)

    # datasets
    def synthesize(self, n, seed, mu=5.0, sigma=1.2, embed_dim=0, max_len=0):
        return Dataset(self, self.L.ref_synthesize(n, mu, sigma, seed, embed_dim, max_len))

    def load_dataset(self, path, limit=-1):
        """load_dataset (dataset.cpp:73-173); raises OracleError with its message."""
        return Dataset(self, self.L.ref_load_dataset(str(path).encode(), limit))

    def save_dataset(self, ds, path):
        if self.L.ref_save_dataset(ds.h, str(path).encode()) != 0:
            raise self._err()

    def samples(self, ds, i):
        out = np.zeros(4096, np.int64)
        k = self.L.ref_dataset_samples(ds.h, C.c_uint64(i), _ptr(out), C.c_int64(4096))
        return out[:k].tolist()

    def from_arrays(self, text, offs, output_len, prompt_len=None, emb=None):
        text = np.ascontiguousarray(text, np.uint8)
        offs = np.ascontiguousarray(offs, np.int64)
        ol = np.ascontiguousarray(output_len, np.int64)
        pl = None if prompt_len is None else np.ascontiguousarray(prompt_len, np.int64)
        e = None if emb is None else np.ascontiguousarray(emb, np.float64)
        return Dataset(self, self.L.ref_dataset_from_arrays(
            _ptr(text), _ptr(offs), _ptr(ol), _ptr(pl), len(offs) - 1, _ptr(e),
            0 if e is None else e.shape[1]))

    def split(self, ds, frac, seed):
        return (Dataset(self, self.L.ref_split(ds.h, frac, seed, 0)),
                Dataset(self, self.L.ref_split(ds.h, frac, seed, 1)))

    def subset(self, ds, idx):
        idx = np.ascontiguousarray(idx, np.int64)
        return Dataset(self, self.L.ref_subset(ds.h, _ptr(idx), len(idx)))

    # predictor
    def extract(self, ex, text: bytes, emb=None):
        cap = max(1, len(text) * 16 + ex.dim)
        idx = np.zeros(cap, np.uint32)
        val = np.zeros(cap, np.float64)
        embc = None if emb is None else np.ascontiguousarray(emb, np.float64)
        n = self.L.ref_extract(C.byref(ex), C.c_char_p(text), C.c_int64(len(text)), _ptr(embc),
                               C.c_int64(0 if emb is None else len(emb)), _ptr(idx), _ptr(val),
                               C.c_int64(cap))
        if n < 0:
            raise self._err()
        return idx[:n].copy(), val[:n].copy()

    def extract_all(self, ex, ds):
        rp = np.zeros(ds.n + 1, np.int64)
        cap = int(ds.offs[-1]) * 2 + ds.n * 4 + 16
        idx = np.zeros(cap, np.uint32)
        val = np.zeros(cap, np.float64)
        tot = self.L.ref_extract_all(C.byref(ex), ds.h, _ptr(rp), _ptr(idx), _ptr(val), cap)
        if tot < 0:
            raise self._err()
        return rp, idx[:tot].copy(), val[:tot].copy()

    def score_batch(self, ex, ds, w, bias=0.0):
        out = np.zeros(ds.n, np.float64)
        rc = self.L.ref_score_batch(C.byref(ex), ds.h, _ptr(np.ascontiguousarray(w, np.float64)),
                                    bias, _ptr(out))
        if rc != 0:
            raise self._err()
        return out

    def evaluate_ranking(self, ex, ds, w, bias=0.0):
        tau = C.c_double()
        counts = np.zeros(5, np.uint64)
        rc = self.L.ref_evaluate_ranking(C.byref(ex), ds.h, _ptr(np.ascontiguousarray(w, np.float64)),
                                         bias, C.byref(tau), _ptr(counts))
        if rc != 0:
            raise self._err()
        return tau.value, counts

    def train(self, ds, ex, objective=0, delta=0.2, margin=1.0, epochs=5, batch=128, lr=0.1,
              seed=0, ppe=100000, lists_per_epoch=2000, list_size=10):
        w = np.zeros(ex.dim, np.float64)
        bias = C.c_double()
        lt = np.zeros(max(epochs, 1), np.float64)
        rc = self.L.ref_train(ds.h, C.byref(ex), objective, delta, margin, epochs, batch, lr,
                              seed, ppe, lists_per_epoch, list_size, _ptr(w), C.byref(bias),
                              _ptr(lt))
        if rc != 0:
            raise self._err()
        return w, bias.value, lt[:epochs].copy()

    def pointwise_order(self, n, seed):
        out = np.zeros(n, np.uint32)
        if self.L.ref_pointwise_order(n, seed, _ptr(out)) != 0:
            raise self._err()
        return out

    def listmle_lists(self, ds, nlists, list_size, seed):
        k = min(list_size, len(ds))
        out = np.zeros(nlists * k, np.uint32)
        if self.L.ref_listmle_lists(ds.h, nlists, list_size, seed, _ptr(out)) != 0:
            raise self._err()
        return out

    def build_pairs(self, ds, delta, max_pairs, seed):
        a = np.zeros(max_pairs, np.uint32)
        b = np.zeros(max_pairs, np.uint32)
        y = np.zeros(max_pairs, np.int32)
        rel = np.zeros(max_pairs, np.float64)
        n = self.L.ref_build_pairs(ds.h, delta, max_pairs, seed, _ptr(a), _ptr(b), _ptr(y), _ptr(rel))
        if n < 0:
            raise self._err()
        return a[:n].copy(), b[:n].copy(), y[:n].copy(), rel[:n].copy()

    def pad_dataset(self, ds, pad_tokens, pad_seed):
        """C4 padding of SURVEY §8(d) applied in place (ref_capi.cpp)."""
        if self.L.ref_pad_dataset(ds.h, pad_tokens, pad_seed) != 0:
            raise self._err()

    def score_order(self, ex, ds, w, bias=0.0):
        """score_batch + select_batch of a burst (ref_capi.cpp ref_score_order)."""
        s = np.zeros(ds.n, np.float64)
        o = np.zeros(ds.n, np.uint64)
        if self.L.ref_score_order(C.byref(ex), ds.h, _ptr(np.ascontiguousarray(w, np.float64)),
                                  bias, _ptr(s), _ptr(o)) != 0:
            raise self._err()
        return s, o.astype(np.int64)

    def select_batch(self, arrival, ids, score, boosted, now, free_slots):
        n = len(arrival)
        arena, offs = ids_arena(ids)
        out = np.zeros(max(n, 1), np.uint64)
        k = self.L.ref_select_batch(C.c_int64(n), _ptr(np.ascontiguousarray(arrival, np.float64)),
                                    C.c_char_p(arena), _ptr(offs),
                                    _ptr(np.ascontiguousarray(score, np.float64)),
                                    _ptr(np.ascontiguousarray(boosted, np.uint8)),
                                    C.c_double(now), C.c_uint64(free_slots), _ptr(out))
        if k < 0:
            raise self._err()
        return out[:k].astype(np.int64)

    def kendall(self, x, y, serial=True):
        tau = C.c_double()
        counts = np.zeros(5, np.uint64)
        rc = self.L.ref_kendall(_ptr(np.ascontiguousarray(x, np.float64)),
                                _ptr(np.ascontiguousarray(y, np.float64)), C.c_int64(len(x)),
                                C.c_int(1 if serial else 0), C.byref(tau), _ptr(counts))
        if rc != 0:
            raise self._err()
        return tau.value, counts

    def poisson(self, ds, rate, seed):
        t = np.zeros(ds.n, np.float64)
        rc = self.L.ref_poisson(ds.h, rate, seed, _ptr(t))
        if rc != 0:
            raise self._err()
        return t

    def simulate(self, ds, arrivals=None, policy="fcfs", ex=None, w=None, bias=0.0,
                 batch_limit=32, starvation_s=120.0):
        pol = {"fcfs": 0, "pars": 1, "oracle": 2, "scores": 3}[policy]
        arr = None if arrivals is None else np.ascontiguousarray(arrivals, np.float64)
        wc = None if w is None else np.ascontiguousarray(w, np.float64)
        h = self.L.ref_simulate(ds.h, _ptr(arr), pol, C.byref(ex) if ex is not None else None,
                                _ptr(wc), bias, batch_limit, starvation_s, 0)
        if not h:
            raise self._err()
        try:
            k = self.L.ref_sim_count(h)
            rec = np.zeros(k, np.int64)
            arrv, adm, fin, ptl = (np.zeros(k, np.float64) for _ in range(4))
            self.L.ref_sim_requests(h, ds.h, _ptr(rec), _ptr(arrv), _ptr(adm), _ptr(fin), _ptr(ptl))
            mean, p90 = C.c_double(), C.c_double()
            self.L.ref_sim_summary(h, C.byref(mean), C.byref(p90))
            return dict(iterations=self.L.ref_sim_iterations(h), seconds=self.L.ref_sim_seconds(h),
                        record=rec, arrival=arrv, admit=adm, finish=fin, ptl=ptl,
                        mean_ms=mean.value, p90_ms=p90.value)
        finally:
            self.L.ref_sim_free(h)


def fnv64_bytes(data: bytes, h: int = 0xCBF29CE484222325) -> int:
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def fnv64_array(a: np.ndarray) -> str:
    """SURVEY Appendix B hash convention: FNV-1a-64 over the little-endian
    8-byte encoding of each value (uint64 indices / raw IEEE doubles)."""
    if a.dtype == np.float64:
        b = a.astype("<f8").tobytes()
    else:
        b = a.astype("<u8").tobytes()
    return f"{fnv64_bytes(b):016x}"


def default_extractor():
    return Extractor.make()
