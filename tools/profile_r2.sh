#!/bin/bash
# Round-2 evidence run ON THE GPU BOX (gpurun): ncu captures of the C4
# kernels (hashing lane kernel + exact chain kernel), the launch list of a
# short bench run, and the integer-issue microbenchmark (roofline peak).
set -u
OUT=${1:-gpurun_out}
mkdir -p $OUT
./tools/micro/int_issue_bin > $OUT/int_issue.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'featurize_lane|chain_slots' -s 4 -c 2 \
  -o $OUT/feat_full -f python bench.py --prompts 200000 --steps 1 --warmup 3 --no-pairs --no-cpu \
  --no-e2e --no-configs > $OUT/ncu_feat.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 \
  > $OUT/ncu_launches.log 2>&1
for f in $OUT/ncu_feat.log $OUT/ncu_launches.log; do tail -n 2 $f; done
