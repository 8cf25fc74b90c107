#!/bin/bash
# Round-2 compute-sanitizer + ThreadSanitizer evidence ON THE GPU BOX
# (gpurun): racecheck and synccheck over the kernels that rely on
# warp-synchronous shared memory (featurize lane kernel, radix sort / merge,
# SGD cluster + CSC build), memcheck over the data-parallel layer, and TSan
# over the drop-in's threaded compare_policies (README burst-500 driver).
# Logs land in $OUT; summarised into profiles/.
set -u
OUT=${1:-gpurun_out/san}
mkdir -p $OUT
: > $OUT/summary.txt
SEL_FEAT="exact_scores_bit_identical or sequential_lane_kernel_random_texts or fast_scores"
SEL_SORT="priority_order_sizes or priority_order_large or merge_shard"
SEL_CSR="features_score or score_records or dp_train or allpairs_matches"
for tool in racecheck synccheck; do
  for grp in FEAT SORT; do
    sel=SEL_$grp
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py \
      -m gpu -q -x -k "${!sel}" > $OUT/${tool}_${grp}.log 2>&1
    echo "$tool $grp rc=$?" >> $OUT/summary.txt
    tail -n 3 $OUT/${tool}_${grp}.log >> $OUT/summary.txt
  done
  # the same featurize tests on the two-kernel (unfused) exact path (the
  # fused kernel's ring hand-off between hashing and chain warps uses
  # shared-memory atomics ordered by fences; both paths are checked)
  PARS_FEAT_UNFUSED=1 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py \
    -m gpu -q -x -k "$SEL_FEAT" > $OUT/${tool}_FEAT_unfused.log 2>&1
  echo "$tool FEAT (unfused) rc=$?" >> $OUT/summary.txt
  tail -n 3 $OUT/${tool}_FEAT_unfused.log >> $OUT/summary.txt
  # the staged CSR gather-dot (pars_dev_features_score) and the DP step around it
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests -m gpu -q -x \
    -k "$SEL_CSR" > $OUT/${tool}_CSR.log 2>&1
  echo "$tool CSR rc=$?" >> $OUT/summary.txt
  tail -n 3 $OUT/${tool}_CSR.log >> $OUT/summary.txt
  # the cluster SGD epoch (csc_build_kernel + sgd_cluster_kernel) at a size
  # racecheck finishes: tools/san_sgd.py
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/san_sgd.py \
    > $OUT/${tool}_SGD.log 2>&1
  echo "$tool SGD rc=$?" >> $OUT/summary.txt
  tail -n 4 $OUT/${tool}_SGD.log >> $OUT/summary.txt
done
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_dp.py -m gpu -q -x \
  > $OUT/memcheck_dp.log 2>&1
echo "memcheck dp rc=$?" >> $OUT/summary.txt
tail -n 3 $OUT/memcheck_dp.log >> $OUT/summary.txt
# ThreadSanitizer: the drop-in's compare_policies runs one std::thread per
# policy over a shared Dataset/trace and one pars_ctx (oracle/Makefile tsan)
TSAN_OPTIONS="halt_on_error=0" timeout 900 ./oracle/_ref/burst500_b200_tsan > $OUT/tsan_b200.out 2> $OUT/tsan_b200.err
echo "tsan burst500_b200 rc=$? warnings=$(grep -c 'WARNING: ThreadSanitizer' $OUT/tsan_b200.err)" >> $OUT/summary.txt
cat $OUT/tsan_b200.out >> $OUT/summary.txt
cat $OUT/summary.txt
