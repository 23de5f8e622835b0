#!/bin/bash
# build_variant.sh NAME SRC "NVCC FLAGS": rebuild one csrc/*.cu with extra -D
# flags and link it with the other release objects into
# build/var/libtxsite_NAME.so (load with TXS_LIB=... for A/B timing).
set -e
cd "$(dirname "$0")/../.."
NAME=$1; SRC=$2; FLAGS=$3
mkdir -p build/var
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc -O3 -std=c++17 -lineinfo $ARCH -Xcompiler -fPIC $FLAGS -c paper_2006_16783_b200/csrc/$SRC.cu -o build/var/$NAME.o
OBJS=$(ls build/*.o | grep -v "/chk_" | grep -v "/$SRC.o")
nvcc $ARCH -shared -o build/var/libtxsite_$NAME.so build/var/$NAME.o $OBJS
echo built build/var/libtxsite_$NAME.so
