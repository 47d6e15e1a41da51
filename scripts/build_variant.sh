#!/bin/bash
# Build lib/libsa_NAME.so with minsum_tc.cu taken from SRC (a csrc directory, e.g. an
# extracted older commit) and every other object from the current in-tree build, for
# A/B runs in one gpurun call (binding.py loads $SA_LIBSA when set).
#   scripts/build_variant.sh NAME SRC_CSRC_DIR [extra nvcc flags]
set -e
cd "$(dirname "$0")/.."
NAME=$1; SRC=$2; shift 2
L=paper_0905_1744_b200/lib
mkdir -p $L/obj_$NAME
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
  -I include "$@" -c $SRC/${TU:-minsum_tc.cu} -o $L/obj_$NAME/${TU:-minsum_tc.cu}.o
objs=$(ls $L/obj/*.o | grep -v ${TU:-minsum_tc.cu}.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static $objs $L/obj_$NAME/${TU:-minsum_tc.cu}.o -ldl -o $L/libsa_$NAME.so
echo "$L/libsa_$NAME.so"
