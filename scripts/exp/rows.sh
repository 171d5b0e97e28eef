set -e
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python bench.py > gpurun_out/bench_lease.json
tail -c 600 gpurun_out/bench_lease.json
