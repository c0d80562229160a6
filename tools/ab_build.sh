#!/bin/bash
# Builds an A/B variant of the library with extra nvcc flags into
# paper_2510_15271_b200/variants/<name>.so (git-ignored; travels to the box).
# usage: tools/ab_build.sh NAME "-DFOO=1 ..."
set -e
NAME=$1; FLAGS=$2
CS=paper_2510_15271_b200/csrc
OUT=paper_2510_15271_b200/variants; mkdir -p $OUT; rm -rf /tmp/ab_$NAME; mkdir -p /tmp/ab_$NAME
NCCL=$(python -c "import nvidia.nccl,os;print(list(nvidia.nccl.__path__)[0])")
for f in $(cd $CS && ls *.cu | sed "s/\.cu$//"); do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$NCCL/include \
       --expt-relaxed-constexpr $FLAGS -c $CS/$f.cu -o /tmp/ab_$NAME/$f.o &
  PIDS="$PIDS $!"
done
for p in $PIDS; do wait $p || { echo "compile failed"; exit 1; }; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/$NAME.so /tmp/ab_$NAME/*.o \
     -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath,$NCCL/lib
echo built $OUT/$NAME.so
