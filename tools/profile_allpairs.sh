#!/bin/bash
# all-pairs (C5) capture + the pair tests, bench and racecheck, ON THE GPU BOX (gpurun)
set -u
OUT=gpurun_out/prof_ap; mkdir -p $OUT
N="ncu --set full --clock-control none --import-source on"
timeout 600 $N -k regex:"allpairs_sorted|tile_sort" -s 2 -c 2 -o $OUT/pairs_full -f python bench.py --prompts 20000 --steps 1 \
  --warmup 3 --no-cpu --no-e2e --no-configs > $OUT/ncu_pairs.log 2>&1
tail -2 $OUT/ncu_pairs.log
python -m pytest tests -m gpu -x -q -k "pair or tau or train or dp" 2>&1 | tail -1
python bench.py --prompts 20000 --no-cpu --no-e2e --no-configs > gpurun_out/b_ap3.log 2>&1
compute-sanitizer --tool racecheck python -m pytest tests -m gpu -x -q -k "allpairs_sorted or pair_plan" 2>&1 | grep -E "RACECHECK|passed|failed" | tail -3
