#!/bin/bash
# Build a tuning variant of the library with extra -D flags:
#   tools/build_variant.sh NAME "-DHPAC_BINO_MIN_CTAS=6 ..."
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; FLAGS=$2
OUT=$ROOT/tools/variants/$NAME; mkdir -p $OUT
for f in $ROOT/paper_2308_16877_b200/csrc/*.cu $ROOT/paper_2308_16877_b200/csrc/*.cpp; do
  b=$(basename $f); b=${b%.*}
  if [ "$b" = engine_team ] || [ ! -f $OUT/$b.o ]; then
    src=$ROOT/paper_2308_16877_b200/build/$b.o
    if [ "$b" != engine_team ] && [ -f $src ]; then cp $src $OUT/$b.o; continue; fi
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I$ROOT/include -I$ROOT/paper_2308_16877_b200/csrc \
      -Xcompiler -fPIC,-fvisibility=hidden $FLAGS -x cu -c $f -o $OUT/$b.o
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libhpac_b200.so $OUT/*.o -lcudart_static -lrt -ldl -lpthread
echo $OUT/libhpac_b200.so
