#!/bin/bash
# Round-2 compute-sanitizer evidence ON THE GPU BOX (gpurun): racecheck and
# synccheck over the kernels that rely on warp-synchronous shared memory
# (featurize lane kernel, radix sort / merge, SGD cluster), memcheck over the
# data-parallel layer. Logs land in $OUT; summarised into profiles/.
set -u
OUT=${1:-gpurun_out/san}
mkdir -p $OUT
SEL_FEAT="exact_scores_bit_identical or sequential_lane_kernel_random_texts or fast_scores"
SEL_SORT="priority_order_sizes or priority_order_large or merge_shard"
SEL_SGD="sgd_epoch_bit_identical"
for tool in racecheck synccheck; do
  for grp in FEAT SORT SGD; do
    sel=SEL_$grp
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py \
      -m gpu -q -x -k "${!sel}" > $OUT/${tool}_${grp}.log 2>&1
    echo "$tool $grp rc=$?" >> $OUT/summary.txt
    tail -n 3 $OUT/${tool}_${grp}.log >> $OUT/summary.txt
  done
done
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_dp.py -m gpu -q -x \
  > $OUT/memcheck_dp.log 2>&1
echo "memcheck dp rc=$?" >> $OUT/summary.txt
tail -n 3 $OUT/memcheck_dp.log >> $OUT/summary.txt
cat $OUT/summary.txt
