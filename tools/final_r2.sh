#!/bin/bash
# Round-2 closing evidence ON THE GPU BOX (gpurun): GPU tests, smoke, the
# bench line (both arms), a one-pass sort capture and the launch list.
# Numbers printed by runs under ncu are never bench values.
set -u
OUT=${1:-gpurun_out/final}
mkdir -p $OUT
python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; tail -n 1 $OUT/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; tail -n 1 $OUT/smoke.log
python bench.py > $OUT/bench.log 2> $OUT/bench.err; tail -n 1 $OUT/bench.log | cut -c1-200
python bench.py --impl reference > $OUT/bench_ref.log 2> $OUT/bench_ref.err; tail -n 1 $OUT/bench_ref.log | cut -c1-200
# one sort call's kernels (the first call of tools/sort_ab.py: burst tie
# ranks, 1 M keys): init, plan, the 4 high-word passes, the fixup, the first
# gated (idle) full-LSD pass
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"radix_" -c 8 \
  -o $OUT/sort_full -f python tools/sort_ab.py > $OUT/ncu_sort.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 \
  > $OUT/ncu_launches.log 2>&1
for f in $OUT/ncu_*.log; do echo "$f: $(tail -n 1 $f | cut -c1-160)"; done
