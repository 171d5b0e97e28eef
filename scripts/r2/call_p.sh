#!/usr/bin/env bash
O=gpurun_out/r2p; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_small.py tests/test_gpu_robustness.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include scripts/r2/host_floor.cu -o /tmp/host_floor \
  -L paper_1506_08503_b200 -l:libgaes_b200.so -Xlinker -rpath=$PWD/paper_1506_08503_b200 > $O/build.log 2>&1
/tmp/host_floor > $O/host_floor.txt 2>&1
/tmp/host_floor > $O/host_floor2.txt 2>&1
python -m paper_1506_08503_b200.sweep --kind count --counts 1,10,100,1000,10000,100000 --out $O/sweep_count_cuda.csv > $O/sweep.log 2>&1
python bench.py --config 1 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err
