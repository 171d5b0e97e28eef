#!/usr/bin/env bash
O=gpurun_out/r2m; mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?" >> $O/rc.txt
python bench.py --config 5 --no-e2e > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "cfg5 rc=$?" >> $O/rc.txt
