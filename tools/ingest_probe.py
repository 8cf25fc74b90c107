"""Where the GPU dataset loader's time goes on the C4 JSONL (1M records,
~2.2 GB, pinned host bytes): the raw H2D copy alone vs the full
pars_load_dataset_bytes call.

    python tools/ingest_probe.py [--records N]
"""
import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2510_03243_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--records", type=int, default=bench.N_PROMPTS)
    args = ap.parse_args()
    import torch
    wl = P.Workload.synthesize(args.records, bench.SEED, pad_tokens=bench.PAD_TOKENS,
                               pad_seed=bench.PAD_SEED)
    n = len(wl)
    parts = [b'{"embedding_dim":0,"format":"pars.dataset","version":1}\n']
    for i in range(n):
        parts.append(b'{"id":"p%07d","output_len":%d,"prompt":"' % (i, int(wl.output_len[i])))
        parts.append(wl.text[wl.offsets[i]:wl.offsets[i + 1]].tobytes())
        parts.append(b'"}\n')
    blob = b"".join(parts)
    nbytes = len(blob)
    L = P.lib()
    hb = C.c_void_p()
    assert L.pars_host_alloc(nbytes, C.byref(hb)) == 0
    host = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(hb.value))
    host[:] = np.frombuffer(blob, np.uint8)
    ctx = P.Context(0)
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    src = torch.from_numpy(host)
    out = {"records": n, "bytes": nbytes}
    ts = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    out["h2d_ms"] = 1e3 * min(ts[1:])
    out["h2d_GBps"] = nbytes / min(ts[1:]) / 1e9
    del dev
    ts = []
    for _ in range(4):
        h = C.c_void_p()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = L.pars_load_dataset_bytes(ctx.h, b"c4.jsonl", C.c_char_p(hb.value), nbytes, -1,
                                       C.byref(h))
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        assert rc == 0, L.pars_last_error()
        L.pars_dataset_free(C.c_void_p(h.value))
    out["load_ms"] = 1e3 * min(ts[1:])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
