timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "tma or rows or cbc" 2>&1 | tail -2
for b in 8 16 64 128; do python scripts/profile_kernels.py cbc_rows 24 $b; done
python scripts/profile_kernels.py cbc_rows 26 64
