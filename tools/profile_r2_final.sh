#!/bin/bash
# Round-2 final evidence run ON THE GPU BOX (gpurun). Captures (ncu --set
# full, one launch each, source-level) of the kernels the bench line reports:
#   feat_full   featurize_lane_kernel<exact, fused> (200k C4 prompts)
#   sort_pass   one radix_onesweep pass over the 1M C4-like keys
#   sgd_full    one C2 sgd_cluster_kernel epoch (782 steps)
#   pairs_full  allpairs_sorted_kernel (C5, 65,536 prompts)
#   dense_full  dense_exact_kernel + dense_fast_kernel (65,536 x 4,096 fp64)
# and the launch list (gpu__time_duration.sum) of a short bench run.
# Numbers printed by runs under ncu are never bench values.
set -u
OUT=${1:-gpurun_out/prof}
mkdir -p $OUT
N="ncu --set full --clock-control none --import-source on"
timeout 600 $N -k regex:featurize_lane -s 3 -c 1 -o $OUT/feat_full -f python tools/feat_ab.py 200000 \
  > $OUT/ncu_feat.log 2>&1
timeout 600 $N -k regex:radix_onesweep -s 20 -c 1 -o $OUT/sort_pass -f python tools/sort_ab.py \
  > $OUT/ncu_sort.log 2>&1
timeout 900 $N -k regex:sgd_cluster_kernel -s 2 -c 1 -o $OUT/sgd_full -f python tools/sgd_ab.py \
  > $OUT/ncu_sgd.log 2>&1
timeout 600 $N -k regex:allpairs_sorted -s 1 -c 1 -o $OUT/pairs_full -f python bench.py --prompts 20000 --steps 1 \
  --warmup 3 --no-cpu --no-e2e --no-configs > $OUT/ncu_pairs.log 2>&1
timeout 600 $N -k regex:dense_ -s 2 -c 2 -o $OUT/dense_full -f python bench.py --prompts 20000 --steps 1 --warmup 3 \
  --no-cpu --no-pairs --no-e2e > $OUT/ncu_dense.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 \
  > $OUT/ncu_launches.log 2>&1
for f in $OUT/ncu_*.log; do echo "$f: $(tail -n 1 $f | cut -c1-200)"; done
