mkdir -p gpurun_out/p5
python tools/feat_ab.py 1000000
timeout 600 ncu --set full --clock-control none --import-source on -k regex:featurize_lane -s 3 -c 1 -o gpurun_out/p5/fused -f python tools/feat_ab.py 200000 > gpurun_out/p5/ncu.log 2>&1
tail -2 gpurun_out/p5/ncu.log
