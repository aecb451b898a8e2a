set -e
ROOT=/root/repo
NAME=$1; FLAGS=$2
OUT=$ROOT/tools/variants/$NAME; mkdir -p $OUT
for f in $ROOT/paper_2308_16877_b200/csrc/*.cu $ROOT/paper_2308_16877_b200/csrc/*.cpp; do b=$(basename $f); b=${b%.*}; cp $ROOT/paper_2308_16877_b200/build/$b.o $OUT/$b.o; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I$ROOT/include -I$ROOT/paper_2308_16877_b200/csrc -Xcompiler -fPIC,-fvisibility=hidden $FLAGS -x cu -c $ROOT/paper_2308_16877_b200/csrc/engine_bs_iact.cu -o $OUT/engine_bs_iact.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libhpac_b200.so $OUT/*.o -lcudart_static -lrt -ldl -lpthread
