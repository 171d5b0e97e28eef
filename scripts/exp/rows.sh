set -e
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for b in 2 4 8 16 64 1024; do echo "bpr=$b"; python scripts/profile_kernels.py cbc_rows 24 $b; done
python scripts/profile_kernels.py cbc_rows 20 64
