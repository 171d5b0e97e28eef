#!/usr/bin/env bash
set -u
O=gpurun_out/r2d; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1506_08503_b200/csrc \
  scripts/r2/small_probe.cu -o /tmp/small_probe -L paper_1506_08503_b200 -l:libgaes_b200.so \
  -Xlinker -rpath=$PWD/paper_1506_08503_b200 > $O/build.log 2>&1
# warm the clocks first
python -c "
import torch,time
x=torch.empty(1<<28,device='cuda',dtype=torch.uint8)
t=time.time()
while time.time()-t<2: x.add_(1)
torch.cuda.synchronize()"
/tmp/small_probe > $O/small_probe.txt 2>&1
/tmp/small_probe > $O/small_probe2.txt 2>&1
python bench.py --config 1 --no-cpu-baseline --no-e2e > $O/bench_cfg1.json 2>$O/bench_cfg1.err
python -m paper_1506_08503_b200.sweep --help > $O/sweep_help.txt 2>&1
