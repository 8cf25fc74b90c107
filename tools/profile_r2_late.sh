#!/bin/bash
# Round-2 late captures ON THE GPU BOX (gpurun): the kernels changed after
# tools/profile_r2_final.sh ran — the SGD cluster epoch (longest-first runs,
# biased counts, 3 chain warps), the staged CSR gather-dot and X^T c.
set -u
OUT=${1:-gpurun_out/prof3}
mkdir -p $OUT
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:sgd_cluster_kernel -s 2 -c 1 -o $OUT/sgd_full -f python tools/sgd_ab.py > $OUT/ncu_sgd.log 2>&1
timeout 600 $N -k regex:cpk_score_coop -s 2 -c 1 -o $OUT/csr_full -f python tools/csr_ab.py > $OUT/ncu_csr.log 2>&1
timeout 600 $N -k regex:xtc_csc -s 2 -c 1 -o $OUT/xtc_full -f python bench.py --prompts 20000 --steps 1 --warmup 3 \
  --no-cpu --no-e2e --no-configs > $OUT/ncu_xtc.log 2>&1
for f in $OUT/ncu_*.log; do echo "$f: $(tail -n 1 $f | cut -c1-160)"; done
