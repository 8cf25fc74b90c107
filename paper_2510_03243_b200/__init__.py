"""B200-native PARS predictor hot path (arXiv 2510.03243).

Scoring (hashed n-gram featurizer + linear head), length-gap-filtered
margin-ranking training, and the SJF priority order — hand-written sm_100a
kernels in libpars_cuda.so behind the C ABI of include/pars_cuda.h. See
DESIGN.md.
"""
from ._lib import (  # noqa: F401
    MODE_EXACT,
    MODE_FAST,
    Context,
    DataParallel,
    Extractor,
    Features,
    ParsError,
    Workload,
    build_pairs,
    dp_shard,
    nccl_unique_id,
    split_weighted,
    device_count,
    ids_arena,
    length_gap_table,
    lib,
    pack_texts,
    pinned_empty,
    tie_ranks,
)

__all__ = [
    "MODE_EXACT", "MODE_FAST", "Context", "DataParallel", "dp_shard", "nccl_unique_id",
    "split_weighted", "Extractor", "Features", "ParsError", "Workload",
    "build_pairs", "device_count", "ids_arena", "length_gap_table", "lib", "pack_texts",
    "pinned_empty", "tie_ranks",
]
