import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2510_03243_b200 as P
ctx = P.Context(0)
g = P.Workload.synthesize(2048, 22)
sel = np.nonzero(g.prompt_len <= 128)[0][:1024]
arena, offs = P.pack_texts([g.text[g.offsets[i]:g.offsets[i+1]].tobytes() for i in sel])
tie = np.arange(len(sel), dtype=np.uint32)
w = np.random.default_rng(1).normal(size=4096)
ex = P.Extractor.make()
outs = (P.pinned_empty(len(sel), np.float64), P.pinned_empty(len(sel), np.int64))
for label, kw in (("pageable", {}), ("pinned", {"out": outs})):
    lat = []
    for k in range(50):
        t0 = time.perf_counter()
        ctx.score_order(ex, arena, offs, w, tie, **kw)
        lat.append(time.perf_counter() - t0)
    print(label, "median ms", 1e3 * float(np.median(lat[5:])))

# fixed overhead: one tiny prompt
a1, o1 = P.pack_texts([b"hello world"])
lat = []
for k in range(50):
    t0 = time.perf_counter()
    ctx.score_order(ex, a1, o1, w, np.zeros(1, np.uint32))
    lat.append(time.perf_counter() - t0)
print("n=1 median ms", 1e3 * float(np.median(lat[5:])))
lat = []
for k in range(50):
    t0 = time.perf_counter()
    ctx.score_text(ex, arena, offs, w)
    lat.append(time.perf_counter() - t0)
print("score_text 1024 median ms", 1e3 * float(np.median(lat[5:])))
