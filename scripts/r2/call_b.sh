#!/usr/bin/env bash
set -u
O=gpurun_out/r2b; mkdir -p $O
python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?" >> $O/rc.txt
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/rc.txt
timeout 2400 python -m pytest tests/test_gpu_multirank.py -x -q > $O/multirank.log 2>&1; echo "multirank rc=$?" >> $O/rc.txt
