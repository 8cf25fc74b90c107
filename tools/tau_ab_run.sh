# tau A/B on the GPU box: tools/tau_ab.py over builds in build_var/ (and the
# in-tree library as "main"), then the GPU tests that touch tau.
mkdir -p gpurun_out/tau
for n in 100000 1000000 10000; do
 for v in ${TAU_VARIANTS:-taubase main}; do
  if [ $v = main ]; then L=""; else L="PARS_CUDA_LIB=build_var/$v/libpars_cuda.so"; fi
  echo "$v $(env $L timeout 300 python tools/tau_ab.py $n 50 2>&1 | tail -1)"
 done
done > gpurun_out/tau/ab.log 2>&1
cat gpurun_out/tau/ab.log
timeout 600 python -m pytest tests -m gpu -q -k "tau or kendall or graph or conformance or acceptance" 2>&1 | tail -2
