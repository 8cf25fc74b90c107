"""ctypes bindings to libpars_cuda.so (include/pars_cuda.h).

This is the Python face of the B200 hot path; the function names and
argument meanings mirror the reference's C++ predictor/scheduler API
(/root/reference/proj/include/pars/*.hpp) so the parity tests read like the
reference's own tests. There is no CPU fallback: if the shared library is
missing or no sm_100 device is present, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

LIB_PATH = Path(os.environ.get("PARS_CUDA_LIB", "") or
                (Path(__file__).resolve().parent / "libpars_cuda.so"))

MODE_EXACT = 0  # PARS_MODE_EXACT_F64
MODE_FAST = 1  # PARS_MODE_FAST_F32


class ParsError(RuntimeError):
    """pars::Error equivalent: carries the library's message verbatim."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class Extractor(C.Structure):
    """pars::FeatureExtractor (features.hpp:17-25)."""

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
    def make(cls, dim: int = 4096, word: Sequence[int] = (1,), char: Sequence[int] = (3,),
             norm: str = "l2", kind: str = "hashed") -> "Extractor":
        e = cls()
        e.kind = 0 if kind in ("hashed", "hashed_text") else 1
        e.dim = dim
        e.norm = 1 if norm == "l2" else 0
        if len(word) > 8 or len(char) > 8:
            raise ValueError("at most 8 word / 8 char n-gram orders")
        e.n_word, e.n_char = len(word), len(char)
        for i, w in enumerate(word):
            e.word[i] = w
        for i, c in enumerate(char):
            e.chr[i] = c
        return e


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = C.CDLL(str(LIB_PATH))
    vp, i64, u64, i32, u32, dbl = C.c_void_p, C.c_int64, C.c_uint64, C.c_int32, C.c_uint32, C.c_double
    sig = {
        "pars_last_error": (C.c_char_p, []),
        "pars_version": (C.c_char_p, []),
        "pars_device_count": (C.c_int, [vp]),
        "pars_ctx_create": (C.c_int, [C.c_int, vp]),
        "pars_ctx_destroy": (None, [vp]),
        "pars_ctx_synchronize": (C.c_int, [vp]),
        "pars_ctx_launches": (u64, [vp]),
        "pars_host_alloc": (C.c_int, [C.c_size_t, vp]),
        "pars_host_free": (None, [vp]),
        "pars_score_text": (C.c_int, [vp, vp, vp, vp, i64, vp, dbl, C.c_int, vp]),
        "pars_dev_score_text": (C.c_int, [vp, vp, vp, vp, i64, vp, dbl, C.c_int, vp, vp]),
        "pars_score_embeddings": (C.c_int, [vp, vp, vp, i64, vp, dbl, C.c_int, vp]),
        "pars_dev_score_embeddings": (C.c_int, [vp, vp, vp, i64, vp, dbl, C.c_int, vp, vp]),
        "pars_kendall_tiles": (i64, [i64]),
        "pars_dev_kendall_counts": (C.c_int, [vp, vp, vp, i64, i64, i64, vp, vp]),
        "pars_kendall_finish": (C.c_int, [vp, i64, vp, vp]),
        "pars_load_dataset": (C.c_int, [vp, C.c_char_p, i64, vp]),
        "pars_load_dataset_bytes": (C.c_int, [vp, C.c_char_p, C.c_char_p, i64, i64, vp]),
        "pars_dataset_size": (i64, [vp]),
        "pars_dataset_text_bytes": (i64, [vp]),
        "pars_dataset_id_bytes": (i64, [vp]),
        "pars_dataset_embedding_dim": (i64, [vp]),
        "pars_dataset_dev_text": (vp, [vp]),
        "pars_dataset_dev_offsets": (vp, [vp]),
        "pars_dataset_dev_output_len": (vp, [vp]),
        "pars_dataset_export": (C.c_int, [vp] * 7),
        "pars_dataset_samples": (i64, [vp, i64, vp, i64]),
        "pars_dataset_free": (None, [vp]),
        "pars_extract": (C.c_int, [vp, vp, vp, vp, i64, vp, vp]),
        "pars_features_upload": (C.c_int, [vp, u32, i64, vp, vp, vp, vp]),
        "pars_features_rows": (i64, [vp]),
        "pars_features_nnz": (i64, [vp]),
        "pars_features_download": (C.c_int, [vp, vp, vp, vp, vp]),
        "pars_features_free": (None, [vp]),
        "pars_features_score": (C.c_int, [vp, vp, vp, dbl, vp]),
        "pars_build_pairs": (i64, [vp, i64, dbl, u64, u64, vp, vp, vp, vp]),
        "pars_length_gap_table": (C.c_int, [dbl, i64, vp]),
        "pars_allpairs": (C.c_int, [vp, vp, vp, i64, dbl, dbl, vp, vp, vp, vp]),
        "pars_allpairs_tiles": (i64, [i64]),
        "pars_allpairs_algo": (C.c_int, [vp, vp, vp, i64, dbl, dbl, C.c_int, vp, vp, vp, vp]),
        "pars_pair_plan_create": (C.c_int, [vp, vp, i64, dbl, vp]),
        "pars_pair_plan_kept": (u64, [vp]),
        "pars_pair_plan_sorted": (C.c_int, [vp]),
        "pars_pair_plan_free": (None, [vp]),
        "pars_dev_allpairs_plan": (C.c_int, [vp, vp, vp, dbl, i64, i64, vp, vp, vp, vp]),
        "pars_dev_allpairs": (C.c_int, [vp, vp, vp, i64, dbl, dbl, i64, i64, i64, vp, vp, vp, vp]),
        "pars_dev_xt_c": (C.c_int, [vp, vp, vp, i64, i64, vp, vp]),
        "pars_pointwise_epoch": (C.c_int, [vp, vp, vp, i64, vp, i32, dbl, vp, vp, vp]),
        "pars_listmle_epoch": (C.c_int, [vp, vp, vp, i64, i32, i32, dbl, vp, dbl, vp]),
        "pars_pointwise_order": (C.c_int, [i64, u64, vp]),
        "pars_listmle_lists": (C.c_int, [vp, vp, vp, i64, i64, i32, u64, vp]),
        "pars_train_baseline": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, i64, i32, i32, i32, dbl, u64,
                                          u64, i32, vp, vp, vp]),
        "pars_sgd_epoch": (C.c_int, [vp, vp, vp, vp, vp, i64, i32, dbl, dbl, vp, dbl, vp, vp]),
        "pars_sgd_epoch_algo": (C.c_int, [vp, vp, vp, vp, vp, i64, i32, dbl, dbl, vp, dbl, vp, vp,
                                          C.c_int]),
        "pars_train_pairwise": (C.c_int, [vp, vp, vp, vp, vp, i64, dbl, dbl, i32, i32, dbl, u64,
                                          u64, vp, vp, vp]),
        "pars_priority_order": (C.c_int, [vp, vp, vp, vp, i64, vp]),
        "pars_dev_features_score": (C.c_int, [vp, vp, i64, i64, vp, dbl, vp, vp]),
        "pars_score_order": (C.c_int, [vp, vp, vp, vp, i64, vp, dbl, C.c_int, vp, vp, vp, vp]),
        "pars_dev_priority_order": (C.c_int, [vp, vp, vp, vp, i64, vp, vp]),
        "pars_tie_ranks": (C.c_int, [vp, vp, vp, i64, vp]),
        "pars_kendall_tau": (C.c_int, [vp, vp, vp, i64, vp, vp]),
        "pars_kendall_tau_algo": (C.c_int, [vp, vp, vp, i64, vp, vp, C.c_int]),
        "pars_dev_merge_orders": (C.c_int, [vp, vp, vp, vp, vp, vp, C.c_int, vp, vp]),
        "pars_dev_kendall_tau": (C.c_int, [vp, vp, vp, i64, vp, vp, vp]),
        "pars_features_dim": (i64, [vp]),
        "pars_score_records": (C.c_int, [vp, vp, vp, vp, i64, vp, dbl, C.c_int, vp]),
        "pars_dev_merge_rank": (C.c_int, [vp, vp, vp, vp, vp, vp, C.c_int, C.c_int, vp, vp]),
        "pars_nccl_get_unique_id": (C.c_int, [vp]),
        "pars_dp_create": (C.c_int, [vp, vp, C.c_int, C.c_int, vp]),
        "pars_dp_create_from_comm": (C.c_int, [vp, vp, vp]),
        "pars_dp_rank": (C.c_int, [vp]),
        "pars_dp_world": (C.c_int, [vp]),
        "pars_dp_destroy": (None, [vp]),
        "pars_dp_shard": (None, [i64, C.c_int, C.c_int, vp, vp]),
        "pars_dp_score_order": (C.c_int, [vp, vp, vp, vp, i64, vp, dbl, C.c_int, vp, vp, vp, vp,
                                          vp]),
        "pars_dp_train_step": (C.c_int, [vp, vp, vp, vp, dbl, dbl, vp, vp, vp, vp, vp]),
        "pars_dp_kendall_tau": (C.c_int, [vp, vp, vp, i64, vp, vp, vp]),
        "pars_split_weighted": (C.c_int, [vp, i64, C.c_int, vp]),
        "pars_pair_plan_tile_split": (C.c_int, [vp, C.c_int, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


_L: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    global _L
    if _L is None:
        _L = _load()
    return _L


def _err(code: int) -> ParsError:
    return ParsError(code, lib().pars_last_error().decode(errors="replace"))


def _check(rc: int):
    if rc < 0:
        raise _err(rc)
    return rc


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def device_count() -> int:
    n = C.c_int(0)
    rc = lib().pars_device_count(C.byref(n))
    return n.value if rc == 0 else 0


# ---- host-side helpers (sequential by construction) --------------------------

def build_pairs(lengths, delta: float, max_pairs: int, seed: int):
    """build_pairs (pairs.cpp:8-36): returns (a, b, y, rel_diff)."""
    lens = _c(lengths, np.int64)
    a = np.zeros(max_pairs, np.uint32)
    b = np.zeros(max_pairs, np.uint32)
    y = np.zeros(max_pairs, np.int32)
    rel = np.zeros(max_pairs, np.float64)
    n = lib().pars_build_pairs(_p(lens), len(lens), delta, max_pairs, seed, _p(a), _p(b), _p(y), _p(rel))
    _check(n)
    return a[:n].copy(), b[:n].copy(), y[:n].copy(), rel[:n].copy()


def length_gap_table(delta: float, max_len: int) -> np.ndarray:
    t = np.zeros(max_len + 1, np.int32)
    _check(lib().pars_length_gap_table(delta, max_len, _p(t)))
    return t


class _PinnedOwner:
    """Keeps a pars_host_alloc block alive for the arrays viewing it."""

    def __init__(self, nbytes: int):
        self.ptr = C.c_void_p()
        _check(lib().pars_host_alloc(max(nbytes, 1), C.byref(self.ptr)))

    def __del__(self):
        if self.ptr and lib is not None:
            lib().pars_host_free(self.ptr)
            self.ptr = C.c_void_p()


def pinned_empty(n: int, dtype) -> np.ndarray:
    """An uninitialised page-locked host array (pars_host_alloc): result
    buffers that the C ABI fills by direct DMA (e.g. score_order's out=)."""
    dt = np.dtype(dtype)
    owner = _PinnedOwner(n * dt.itemsize)
    buf = (C.c_uint8 * max(n * dt.itemsize, 1)).from_address(owner.ptr.value)
    buf._owner = owner  # the ctypes buffer keeps the allocation alive
    return np.frombuffer(buf, dtype=dt, count=n)


def ids_arena(ids):
    bs = [i.encode() if isinstance(i, str) else bytes(i) for i in ids]
    offs = np.zeros(len(bs) + 1, np.int64)
    offs[1:] = np.cumsum([len(b) for b in bs])
    return np.frombuffer(b"".join(bs) + b"\0", np.uint8).copy(), offs


def tie_ranks(arrival, ids) -> np.ndarray:
    arena, offs = ids_arena(ids)
    arr = _c(arrival, np.float64)
    r = np.zeros(len(arr), np.uint32)
    _check(lib().pars_tie_ranks(_p(arr), _p(arena), _p(offs), len(arr), _p(r)))
    return r


WORKLOAD_LIB_PATH = Path(__file__).resolve().parents[1] / "tools" / "libpars_workload.so"
_WL = None


def workload_lib():
    """The synthetic-workload TOOL library (tools/libpars_workload.so): input
    generation for benchmarks and tests, not part of libpars_cuda.so."""
    global _WL
    if _WL is None:
        if not WORKLOAD_LIB_PATH.exists():
            raise FileNotFoundError(f"{WORKLOAD_LIB_PATH} not built (make -C tools/workload)")
        L = C.CDLL(str(WORKLOAD_LIB_PATH))
        vp, i64 = C.c_void_p, C.c_int64
        for name, res, args in (
                ("pars_workload_synthesize", C.c_int,
                 [C.c_uint64, C.c_double, C.c_double, C.c_uint64, i64, C.c_uint64, vp]),
                ("pars_workload_synthesize_pad", C.c_int,
                 [C.c_uint64, C.c_double, C.c_double, C.c_uint64, i64, C.c_uint64, C.c_int, vp]),
                ("pars_workload_count", i64, [vp]), ("pars_workload_text_bytes", i64, [vp]),
                ("pars_workload_text", vp, [vp]), ("pars_workload_offsets", vp, [vp]),
                ("pars_workload_output_len", vp, [vp]), ("pars_workload_prompt_len", vp, [vp]),
                ("pars_workload_free", None, [vp]), ("pars_workload_last_error", C.c_char_p, []),
                ("pars_workload_token_stats", C.c_int, [vp, vp, i64, vp])):
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _WL = L
    return _WL


@dataclass
class Workload:
    """Synthetic prompts (dataset.cpp:204-297 restated on the host by the
    workload tool library, tools/libpars_workload.so)."""

    text: np.ndarray  # uint8 view of the (pinned) arena
    offsets: np.ndarray
    output_len: np.ndarray
    prompt_len: np.ndarray
    _h: int = 0

    @classmethod
    def synthesize(cls, n: int, seed: int, mu: float = 5.0, sigma: float = 1.2,
                   pad_tokens: int = 0, pad_seed: int = 5, pad_words: str = "filler") -> "Workload":
        """pad_words: "filler" (C4: " w<k>") or "random6" (the C4 hard variant)."""
        L = workload_lib()
        h = C.c_void_p()
        kind = {"filler": 0, "random6": 1}[pad_words]
        rc = L.pars_workload_synthesize_pad(n, mu, sigma, seed, pad_tokens, pad_seed, kind, C.byref(h))
        if rc != 0:
            raise ParsError(rc, L.pars_workload_last_error().decode("utf-8", "replace"))
        cnt = L.pars_workload_count(h)
        nb = L.pars_workload_text_bytes(h)
        text = np.ctypeslib.as_array(C.cast(L.pars_workload_text(h), C.POINTER(C.c_uint8)),
                                     shape=(max(nb, 1),))[:nb]
        offs = np.ctypeslib.as_array(C.cast(L.pars_workload_offsets(h), C.POINTER(C.c_int64)),
                                     shape=(cnt + 1,)).copy()
        ol = np.ctypeslib.as_array(C.cast(L.pars_workload_output_len(h), C.POINTER(C.c_int64)),
                                   shape=(cnt,)).copy()
        pl = np.ctypeslib.as_array(C.cast(L.pars_workload_prompt_len(h), C.POINTER(C.c_int64)),
                                   shape=(cnt,)).copy()
        return cls(text, offs, ol, pl, h.value)

    def __len__(self):
        return len(self.output_len)

    def token_stats(self, b: int = 0, e: Optional[int] = None):
        """(tokens, sum of token lengths, sum of max(0, len - 2), text bytes)
        of prompts [b, e) — the host-side count behind the featurize
        kernel's integer-issue roofline."""
        e = len(self) if e is None else e
        out = np.zeros(4, np.uint64)
        offs = np.ascontiguousarray(self.offsets[b:e + 1])
        workload_lib().pars_workload_token_stats(self.text.ctypes.data, offs.ctypes.data, e - b,
                                                 out.ctypes.data)
        return tuple(int(x) for x in out)

    def prompt(self, i) -> bytes:
        return self.text[self.offsets[i]:self.offsets[i + 1]].tobytes()

    def close(self):
        if self._h:
            workload_lib().pars_workload_free(C.c_void_p(self._h))
            self._h = 0
            self.text = np.zeros(0, np.uint8)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pack_texts(texts: Sequence[bytes]):
    """Concatenate prompt strings into (arena uint8, offsets int64[n+1])."""
    bs = [t.encode() if isinstance(t, str) else bytes(t) for t in texts]
    offs = np.zeros(len(bs) + 1, np.int64)
    offs[1:] = np.cumsum([len(b) for b in bs])
    arena = np.frombuffer(b"".join(bs), np.uint8).copy() if bs else np.zeros(0, np.uint8)
    if arena.size == 0:
        arena = np.zeros(1, np.uint8)
    return arena, offs


class Features:
    """Device-resident CSR produced by extract_all (pars_features*)."""

    def __init__(self, ctx: "Context", handle: int, dim: int):
        self.ctx, self.h, self.dim = ctx, handle, dim

    @property
    def rows(self) -> int:
        return lib().pars_features_rows(C.c_void_p(self.h))

    @property
    def nnz(self) -> int:
        return lib().pars_features_nnz(C.c_void_p(self.h))

    def download(self):
        rows, nnz = self.rows, self.nnz
        rp = np.zeros(rows + 1, np.int64)
        idx = np.zeros(max(nnz, 1), np.uint32)
        val = np.zeros(max(nnz, 1), np.float64)
        _check(lib().pars_features_download(self.ctx.h, C.c_void_p(self.h), _p(rp), _p(idx), _p(val)))
        return rp, idx[:nnz], val[:nnz]

    def score(self, weights, bias: float = 0.0) -> np.ndarray:
        out = np.zeros(self.rows, np.float64)
        _check(lib().pars_features_score(self.ctx.h, C.c_void_p(self.h), _p(_c(weights, np.float64)),
                                         bias, _p(out)))
        return out

    def free(self):
        if self.h:
            lib().pars_features_free(C.c_void_p(self.h))
            self.h = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class GpuDataset:
    """A dataset loaded by the GPU loader (pars_dataset*): device arena +
    offsets (dev_text / dev_offsets for pars_dev_score_text), host exports."""

    def __init__(self, handle: int):
        L = lib()
        self.h = handle
        self.n = L.pars_dataset_size(C.c_void_p(handle))
        self.embedding_dim = L.pars_dataset_embedding_dim(C.c_void_p(handle))

    def __len__(self):
        return self.n

    @property
    def dev_text(self) -> int:
        return lib().pars_dataset_dev_text(C.c_void_p(self.h)) or 0

    @property
    def dev_offsets(self) -> int:
        return lib().pars_dataset_dev_offsets(C.c_void_p(self.h)) or 0

    def export(self):
        """(text uint8, offsets int64[n+1], output_len, prompt_len, ids list)"""
        L, hv = lib(), C.c_void_p(self.h)
        text = np.zeros(max(1, L.pars_dataset_text_bytes(hv)), np.uint8)
        idb = np.zeros(max(1, L.pars_dataset_id_bytes(hv)), np.uint8)
        offs = np.zeros(self.n + 1, np.int64)
        ido = np.zeros(self.n + 1, np.int64)
        ol = np.zeros(max(1, self.n), np.int64)
        pl = np.zeros(max(1, self.n), np.int64)
        _check(L.pars_dataset_export(hv, _p(text), _p(offs), _p(ol), _p(pl), _p(idb), _p(ido)))
        ids = [idb[ido[i]:ido[i + 1]].tobytes().decode("utf-8", "surrogateescape")
               for i in range(self.n)]
        return text[:offs[-1]], offs, ol[:self.n], pl[:self.n], ids

    def samples(self, i: int):
        out = np.zeros(4096, np.int64)
        k = lib().pars_dataset_samples(C.c_void_p(self.h), i, _p(out), 4096)
        return out[:k].tolist()

    def free(self):
        if self.h:
            lib().pars_dataset_free(C.c_void_p(self.h))
            self.h = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class PairPlan:
    """Per-dataset plan of the length-sorted all-pairs kernel (pars_pair_plan*)."""

    def __init__(self, ctx: "Context", lengths, delta: float):
        L = _c(lengths, np.int64)
        h = C.c_void_p()
        _check(lib().pars_pair_plan_create(ctx.h, _p(L), len(L), delta, C.byref(h)))
        self.ctx, self.h, self.n, self.delta = ctx, h.value, len(L), delta

    @property
    def kept(self) -> int:
        return lib().pars_pair_plan_kept(C.c_void_p(self.h))

    @property
    def sorted(self) -> bool:
        return bool(lib().pars_pair_plan_sorted(C.c_void_p(self.h)))

    def run(self, d_scores: int, margin: float, t0: int, t1: int, d_coeff: int, d_counters: int,
            d_partials: int, stream: int = 0):
        _check(lib().pars_dev_allpairs_plan(self.ctx.h, C.c_void_p(self.h), d_scores, margin, t0,
                                            t1, d_coeff, d_counters, d_partials, stream or None))

    def tile_split(self, world: int) -> np.ndarray:
        """Cost-balanced contiguous split of the tile list over `world` ranks
        (pars_pair_plan_tile_split): bounds[world + 1]."""
        b = np.zeros(world + 1, np.int64)
        _check(lib().pars_pair_plan_tile_split(C.c_void_p(self.h), world, _p(b)))
        return b

    def free(self):
        if self.h:
            lib().pars_pair_plan_free(C.c_void_p(self.h))
            self.h = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Context:
    """One CUDA device + its scratch (pars_ctx*)."""

    def __init__(self, device: int = 0):
        L = lib()
        h = C.c_void_p()
        _check(L.pars_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            lib().pars_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return lib().pars_ctx_launches(self.h)

    def synchronize(self):
        _check(lib().pars_ctx_synchronize(self.h))

    # -- scoring ---------------------------------------------------------------
    def score_text(self, ex: Extractor, text: np.ndarray, offsets: np.ndarray, weights,
                   bias: float = 0.0, mode: int = MODE_EXACT, out=None) -> np.ndarray:
        """Scorer::score_batch over prompts given as an arena + offsets.
        out: optional caller-owned float64[n] (page-locked: direct DMA)."""
        offs = _c(offsets, np.int64)
        n = len(offs) - 1
        if out is None:
            out = np.zeros(max(n, 0), np.float64)
        else:
            assert out.dtype == np.float64 and out.flags.c_contiguous and len(out) >= n
        t = text if isinstance(text, np.ndarray) else np.frombuffer(bytes(text), np.uint8)
        _check(lib().pars_score_text(self.h, C.byref(ex), _p(t), _p(offs), n,
                                     _p(_c(weights, np.float64)), bias, mode, _p(out)))
        return out

    def score_order(self, ex: Extractor, text: np.ndarray, offsets: np.ndarray, weights,
                    tie_rank, boosted=None, bias: float = 0.0, mode: int = MODE_EXACT, out=None):
        """enqueue + select_batch in one call: (scores, full admission order).
        out: optional caller-owned (scores float64[n], order int64[n]) arrays,
        reused across calls by a serving loop."""
        offs = _c(offsets, np.int64)
        n = len(offs) - 1
        if out is None:
            scores = np.zeros(max(n, 0), np.float64)
            order = np.zeros(max(n, 0), np.int64)
        else:
            scores, order = out
            assert scores.dtype == np.float64 and order.dtype == np.int64
            assert len(scores) >= n and len(order) >= n
            assert scores.flags.c_contiguous and order.flags.c_contiguous
        t = text if isinstance(text, np.ndarray) else np.frombuffer(bytes(text), np.uint8)
        bst = None if boosted is None else _c(boosted, np.uint8)
        _check(lib().pars_score_order(self.h, C.byref(ex), _p(t), _p(offs), n,
                                      _p(_c(weights, np.float64)), bias, mode,
                                      _p(_c(tie_rank, np.uint32)), _p(bst), _p(scores), _p(order)))
        return scores, order

    def score_texts(self, ex: Extractor, texts: Sequence[bytes], weights, bias=0.0,
                    mode=MODE_EXACT) -> np.ndarray:
        arena, offs = pack_texts(texts)
        return self.score_text(ex, arena, offs, weights, bias, mode)

    def dev_score_text(self, ex: Extractor, d_text: int, d_offsets: int, n: int, d_weights: int,
                       bias: float, mode: int, d_scores: int, stream: int = 0):
        _check(lib().pars_dev_score_text(self.h, C.byref(ex), d_text, d_offsets, n, d_weights,
                                         bias, mode, d_scores, stream or None))

    def score_embeddings(self, ex: Extractor, X, weights, bias=0.0, mode=MODE_EXACT):
        X = _c(X, np.float64)
        out = np.zeros(X.shape[0], np.float64)
        _check(lib().pars_score_embeddings(self.h, C.byref(ex), _p(X), X.shape[0],
                                           _p(_c(weights, np.float64)), bias, mode, _p(out)))
        return out

    # -- features ------------------------------------------------------------
    def extract(self, ex: Extractor, text: np.ndarray, offsets: np.ndarray,
                embeddings=None) -> Features:
        """extract_all (features.cpp:124-141) -> device CSR."""
        offs = _c(offsets, np.int64)
        emb = None if embeddings is None else _c(embeddings, np.float64)
        h = C.c_void_p()
        _check(lib().pars_extract(self.h, C.byref(ex), _p(text), _p(offs), len(offs) - 1, _p(emb),
                                  C.byref(h)))
        return Features(self, h.value, ex.dim)

    def extract_texts(self, ex: Extractor, texts: Sequence[bytes]) -> Features:
        arena, offs = pack_texts(texts)
        return self.extract(ex, arena, offs)

    def upload_features(self, dim: int, row_ptr, idx, val) -> Features:
        rp = _c(row_ptr, np.int64)
        h = C.c_void_p()
        _check(lib().pars_features_upload(self.h, dim, len(rp) - 1, _p(rp),
                                          _p(_c(idx, np.uint32)), _p(_c(val, np.float64)),
                                          C.byref(h)))
        return Features(self, h.value, dim)

    # -- pairs / training ----------------------------------------------------
    def allpairs(self, scores, lengths, delta: float = 0.2, margin: float = 1.0,
                 algo: str = "sorted"):
        """All-pairs margin ranking loss: (coeff int32[n], kept, active, loss_sum).
        algo: "sorted" (length-sorted plan, default) or "general" (unsorted tiles)."""
        s = _c(scores, np.float64)
        L = _c(lengths, np.int64)
        c = np.zeros(len(s), np.int32)
        kept, act, loss = C.c_uint64(), C.c_uint64(), C.c_double()
        _check(lib().pars_allpairs_algo(self.h, _p(s), _p(L), len(s), delta, margin,
                                        0 if algo == "sorted" else 1, _p(c), C.byref(kept),
                                        C.byref(act), C.byref(loss)))
        return c, kept.value, act.value, loss.value

    def load_dataset(self, path, limit: int = -1) -> "GpuDataset":
        """load_dataset (dataset.cpp:73-173) with the records parsed on the GPU."""
        h = C.c_void_p()
        _check(lib().pars_load_dataset(self.h, str(path).encode(), limit, C.byref(h)))
        return GpuDataset(h.value)

    def load_dataset_bytes(self, data: bytes, path: str = "<bytes>", limit: int = -1) -> "GpuDataset":
        h = C.c_void_p()
        _check(lib().pars_load_dataset_bytes(self.h, path.encode(), data, len(data), limit,
                                             C.byref(h)))
        return GpuDataset(h.value)

    def pair_plan(self, lengths, delta: float = 0.2) -> "PairPlan":
        return PairPlan(self, lengths, delta)

    def sgd_epoch(self, feats: Features, a, b, y, batch: int, lr: float, margin: float, w,
                  bias: float = 0.0, algo: str = "auto"):
        """One pairwise SGD epoch (train.cpp:154-166). algo: "auto", "cluster"
        (8-CTA cluster kernel) or "single" (one persistent CTA)."""
        w = np.array(w, np.float64, copy=True)
        a, b, y = _c(a, np.uint32), _c(b, np.uint32), _c(y, np.int32)
        el, act = C.c_double(), C.c_uint64()
        code = {"auto": 0, "cluster": 1, "single": 2}[algo]
        _check(lib().pars_sgd_epoch_algo(self.h, C.c_void_p(feats.h), _p(a), _p(b), _p(y), len(a),
                                         batch, lr, margin, _p(w), bias, C.byref(el),
                                         C.byref(act), code))
        return w, el.value, act.value

    def train_pairwise(self, ex: Extractor, text, offsets, lengths, delta=0.2, margin=1.0,
                       epochs=5, batch=128, lr=0.1, seed=0, pairs_per_epoch=100000):
        """train() with Objective::Pairwise (train.cpp:122-216)."""
        offs = _c(offsets, np.int64)
        lens = _c(lengths, np.int64)
        w = np.zeros(ex.dim, np.float64)
        bias = C.c_double()
        lt = np.zeros(max(epochs, 1), np.float64)
        _check(lib().pars_train_pairwise(self.h, C.byref(ex), _p(text), _p(offs), _p(lens),
                                         len(offs) - 1, delta, margin, epochs, batch, lr, seed,
                                         pairs_per_epoch, _p(w), C.byref(bias), _p(lt)))
        return w, bias.value, lt[:epochs].copy()

    def pointwise_epoch(self, feats: Features, order, target, batch: int, lr: float, w,
                        bias: float = 0.0):
        """One PointwiseL1 epoch (train.cpp:168-183): (w, bias, loss_sum)."""
        w = np.array(w, np.float64, copy=True)
        order, target = _c(order, np.uint32), _c(target, np.float64)
        b, el = C.c_double(bias), C.c_double()
        _check(lib().pars_pointwise_epoch(self.h, C.c_void_p(feats.h), _p(order), len(order),
                                          _p(target), batch, lr, _p(w), C.byref(b), C.byref(el)))
        return w, b.value, el.value

    def listmle_epoch(self, feats: Features, lists, k: int, batch: int, lr: float, w,
                      bias: float = 0.0):
        """One ListwiseListMLE epoch (train.cpp:185-205): (w, loss_sum)."""
        w = np.array(w, np.float64, copy=True)
        lists = _c(lists, np.uint32)
        el = C.c_double()
        _check(lib().pars_listmle_epoch(self.h, C.c_void_p(feats.h), _p(lists), len(lists) // k,
                                        k, batch, lr, _p(w), bias, C.byref(el)))
        return w, el.value

    def train_baseline(self, ex: Extractor, text, offsets, lengths, ids, objective: str,
                       epochs=5, batch=128, lr=0.1, seed=0, lists_per_epoch=2000, list_size=10):
        """train() with Objective::PointwiseL1 ("pointwise_l1") or
        ListwiseListMLE ("listwise_listmle") (train.cpp:122-216)."""
        obj = {"pointwise_l1": 1, "listwise_listmle": 2}[objective]
        offs = _c(offsets, np.int64)
        lens = _c(lengths, np.int64)
        bs = [i.encode() if isinstance(i, str) else bytes(i) for i in ids]
        id_offs = np.zeros(len(bs) + 1, np.int64)
        id_offs[1:] = np.cumsum([len(x) for x in bs])
        arena = np.frombuffer(b"".join(bs) + b"\0", np.uint8)
        w = np.zeros(ex.dim, np.float64)
        bias = C.c_double()
        lt = np.zeros(max(epochs, 1), np.float64)
        _check(lib().pars_train_baseline(self.h, C.byref(ex), _p(text), _p(offs), _p(lens),
                                         _p(arena), _p(id_offs), len(offs) - 1, obj, epochs, batch,
                                         lr, seed, lists_per_epoch, list_size, _p(w),
                                         C.byref(bias), _p(lt)))
        return w, bias.value, lt[:epochs].copy()

    # -- scheduling / metrics ------------------------------------------------
    def priority_order(self, scores, tie_rank, boosted=None) -> np.ndarray:
        """select_batch's full admission order (scheduler.cpp:33-60)."""
        s = _c(scores, np.float64)
        t = _c(tie_rank, np.uint32)
        bst = None if boosted is None else _c(boosted, np.uint8)
        out = np.zeros(len(s), np.int64)
        _check(lib().pars_priority_order(self.h, _p(s), _p(bst), _p(t), len(s), _p(out)))
        return out

    def score_records(self, ex: Extractor, texts, weights, bias: float = 0.0,
                      mode: int = MODE_EXACT) -> np.ndarray:
        """Scorer::score_batch over separate host strings (pars_score_records)."""
        bufs = [t if isinstance(t, bytes) else bytes(t) for t in texts]
        ptrs = (C.c_char_p * max(1, len(bufs)))(*bufs)
        lens = np.array([len(t) for t in bufs], np.int64)
        w = _c(weights, np.float64)
        out = np.zeros(len(bufs), np.float64)
        _check(lib().pars_score_records(self.h, C.byref(ex), ptrs, _p(lens), len(bufs), _p(w), bias,
                                        mode, _p(out)))
        return out

    def kendall_tau(self, x, y, algo: str = "auto"):
        """kendall_tau_b (metrics.cpp:42-64): (tau_b, counts[n_c,n_d,n0,n1,n2]).
        algo: "auto" (sorted unless an input is inf/NaN), "sorted" (O(n log n))
        or "pairs" (all-pairs tiles)."""
        x, y = _c(x, np.float64), _c(y, np.float64)
        counts = np.zeros(5, np.uint64)
        tau = C.c_double()
        code = {"auto": 0, "sorted": 1, "pairs": 2}[algo]
        _check(lib().pars_kendall_tau_algo(self.h, _p(x), _p(y), len(x), _p(counts), C.byref(tau),
                                           code))
        return tau.value, counts

    def dev_kendall_tau(self, d_x: int, d_y: int, n: int, stream=None):
        """kendall_tau_b of device arrays (pointers), stream-ordered."""
        counts = np.zeros(5, np.uint64)
        tau = C.c_double()
        _check(lib().pars_dev_kendall_tau(self.h, d_x, d_y, n, _p(counts), C.byref(tau), stream))
        return tau.value, counts


def split_weighted(weights, world: int) -> np.ndarray:
    """pars_split_weighted (host only): bounds[world + 1] of a contiguous
    split with equal weight per rank."""
    w = _c(weights, np.int64)
    b = np.zeros(world + 1, np.int64)
    _check(lib().pars_split_weighted(_p(w), len(w), world, _p(b)))
    return b


def dp_shard(n: int, world: int, rank: int):
    b, e = C.c_int64(), C.c_int64()
    lib().pars_dp_shard(n, world, rank, C.byref(b), C.byref(e))
    return b.value, e.value


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().pars_nccl_get_unique_id(buf))
    return bytes(buf)


class DataParallel:
    """One rank of the NCCL data-parallel layer (pars_dp*).

    Create on every rank with the same 128-byte unique id (from
    nccl_unique_id() on rank 0, broadcast by the caller) — or wrap an
    existing ncclComm_t with from_comm. Every method is collective."""

    def __init__(self, ctx: "Context", uid: bytes, world: int, rank: int):
        h = C.c_void_p()
        idb = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().pars_dp_create(ctx.h, idb, world, rank, C.byref(h)))
        self.ctx, self.h = ctx, h

    @classmethod
    def from_comm(cls, ctx: "Context", comm_ptr: int) -> "DataParallel":
        self = cls.__new__(cls)
        h = C.c_void_p()
        _check(lib().pars_dp_create_from_comm(ctx.h, C.c_void_p(comm_ptr), C.byref(h)))
        self.ctx, self.h = ctx, h
        return self

    @property
    def rank(self) -> int:
        return lib().pars_dp_rank(self.h)

    @property
    def world(self) -> int:
        return lib().pars_dp_world(self.h)

    def score_order(self, ex: Extractor, d_text: int, d_offsets: int, n_total: int, d_w: int,
                    bias: float, mode: int, d_scores_all: int, d_order_all: int,
                    d_boosted_all: int = 0, d_tie_all: int = 0, stream: int = 0):
        """pars_dp_score_order on device pointers (this rank's shard text)."""
        _check(lib().pars_dp_score_order(self.h, C.byref(ex), d_text, d_offsets, n_total, d_w, bias,
                                         mode, d_boosted_all or None, d_tie_all or None,
                                         d_scores_all or None, d_order_all or None, stream or None))

    def train_step(self, feats: "Features", plan: "PairPlan", d_w: int, margin: float, lr: float,
                   d_coeff: int, d_scores_all: int = 0, d_counters: int = 0, d_loss: int = 0,
                   stream: int = 0):
        """pars_dp_train_step: one full-batch all-pairs step, w updated in place."""
        _check(lib().pars_dp_train_step(self.h, C.c_void_p(feats.h), C.c_void_p(plan.h), d_w, margin,
                                        lr, d_scores_all or None, d_coeff, d_counters or None,
                                        d_loss or None, stream or None))

    def kendall_tau(self, d_x: int, d_y: int, n: int, stream: int = 0):
        counts = np.zeros(5, np.uint64)
        tau = C.c_double()
        _check(lib().pars_dp_kendall_tau(self.h, d_x, d_y, n, _p(counts), C.byref(tau),
                                         stream or None))
        return tau.value, counts

    def close(self):
        if self.h:
            lib().pars_dp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
