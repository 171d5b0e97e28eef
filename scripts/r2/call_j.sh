#!/usr/bin/env bash
O=gpurun_out/r2j; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include scripts/r2/host_floor.cu -o /tmp/host_floor \
  -L paper_1506_08503_b200 -l:libgaes_b200.so -Xlinker -rpath=$PWD/paper_1506_08503_b200 > $O/build.log 2>&1
/tmp/host_floor > $O/host_floor.txt 2>&1
/tmp/host_floor > $O/host_floor2.txt 2>&1
