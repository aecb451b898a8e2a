#!/bin/bash
# Build a tuning variant of the library with extra -D flags, recompiling only
# the listed sources (default engine_team) and reusing the in-tree objects:
#   tools/build_variant.sh NAME "-DHPAC_BINO_MIN_CTAS=6 ..." [engine_thread engine_team ...]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; FLAGS=$2; shift 2
REBUILD=${*:-engine_team}
OUT=$ROOT/tools/variants/$NAME; mkdir -p $OUT
for f in $ROOT/paper_2308_16877_b200/csrc/*.cu $ROOT/paper_2308_16877_b200/csrc/*.cpp; do
  b=$(basename $f); b=${b%.*}
  if [[ " $REBUILD " == *" $b "* ]]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I$ROOT/include -I$ROOT/paper_2308_16877_b200/csrc \
      -Xcompiler -fPIC,-fvisibility=hidden $FLAGS -x cu -c $f -o $OUT/$b.o
  else
    cp $ROOT/paper_2308_16877_b200/build/$b.o $OUT/$b.o
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libhpac_b200.so $OUT/*.o -lcudart_static -lrt -ldl -lpthread
echo $OUT/libhpac_b200.so
