#!/bin/bash
# A/B builds: libpars_cuda.so with one translation unit swapped or rebuilt
# with extra flags, into build_var/NAME/ (git-ignored; travels with gpurun).
# Select it at run time with PARS_CUDA_LIB=build_var/NAME/libpars_cuda.so.
#   tools/build_variant.sh NAME UNIT SRC [nvcc flags...]
#   e.g. tools/build_variant.sh base featurize <(git show HEAD:paper_2510_03243_b200/csrc/featurize.cu)
set -e
NAME=$1; UNIT=$2; SRC=$3; shift 3
ROOT=$(cd "$(dirname "$0")/.." && pwd)
PKG=$ROOT/paper_2510_03243_b200
OUT=$ROOT/build_var/$NAME
JSON_DIR=/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
mkdir -p $OUT
cp "$SRC" $OUT/$UNIT.cu
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ccbin /usr/bin/g++ \
  -Xcompiler -fPIC -Xcompiler -ffp-contract=off -I$ROOT/include -I$PKG/csrc -I$JSON_DIR "$@" \
  -c $OUT/$UNIT.cu -o $OUT/$UNIT.o
OBJS=$(ls $PKG/build/*.o | grep -v "/$UNIT.o$" | grep -v "/shim_")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ -o $OUT/libpars_cuda.so \
  $OBJS $OUT/$UNIT.o -lcudart_static -lrt -lpthread -ldl
echo "$OUT/libpars_cuda.so"
