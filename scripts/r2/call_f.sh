#!/usr/bin/env bash
set -u
O=gpurun_out/r2f; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
python bench.py --config 1 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err; echo "cfg1 rc=$?" >> $O/rc.txt
python bench.py --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo "cfg3 rc=$?" >> $O/rc.txt
python -m paper_1506_08503_b200.sweep --kind count --counts 1,10,100,1000,10000,65536,100000,1000000 --out $O/sweep_count_cuda.csv > $O/sweep.log 2>&1; echo "sweep rc=$?" >> $O/rc.txt
python -m paper_1506_08503_b200.sweep --kind count --device-resident --counts 1,10,100,1000,10000,65536,100000,1000000 --out $O/sweep_count_dev.csv >> $O/sweep.log 2>&1; echo "sweep2 rc=$?" >> $O/rc.txt
