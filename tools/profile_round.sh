#!/bin/bash
# Run ON THE GPU BOX (gpurun): ncu evidence for the bench's kernels.
#  1. --set full capture of the featurize kernel (200k C4 prompts, one launch)
#  2. --set full capture of the all-pairs kernel (C5)
#  3. the launch list (gpu__time_duration.sum) of a short bench run
# Outputs land in gpurun_out/ and are summarised here by tools/ncu_summary.py,
# tools/launch_summary.py and tools/ncu_to_json.py.
set -u
OUT=${1:-gpurun_out}
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:featurize_seq -s 2 -c 1 \
  -o $OUT/feat_full -f python bench.py --prompts 200000 --steps 1 --warmup 3 --no-pairs --no-cpu \
  --no-e2e --no-configs > $OUT/ncu_feat.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:allpairs -s 1 -c 1 \
  -o $OUT/pairs_full -f python bench.py --prompts 20000 --steps 1 --warmup 3 --no-cpu --no-e2e \
  --no-configs > $OUT/ncu_pairs.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_exact -s 1 -c 1 \
  -o $OUT/dense_full -f python bench.py --prompts 20000 --steps 1 --warmup 3 --no-cpu --no-pairs \
  --no-e2e > $OUT/ncu_dense.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 \
  > $OUT/ncu_launches.log 2>&1
for f in $OUT/ncu_feat.log $OUT/ncu_pairs.log $OUT/ncu_launches.log; do tail -n 2 $f; done
