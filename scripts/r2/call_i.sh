#!/usr/bin/env bash
set -u
O=gpurun_out/r2i; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include scripts/r2/host_floor.cu -o /tmp/host_floor \
  -L paper_1506_08503_b200 -l:libgaes_b200.so -Xlinker -rpath=$PWD/paper_1506_08503_b200 > $O/build.log 2>&1
for t in "" "NT=0" "SMALL_BLOCKS_PER_SM=0" "SMALL_ZEROCOPY_KB=0"; do
  echo "== GAES_TUNE=$t" >> $O/host_floor.txt
  GAES_TUNE=$t /tmp/host_floor >> $O/host_floor.txt 2>&1
done
python bench.py --config 1 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err
