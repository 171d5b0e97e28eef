timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cbc or rows or grid or property or out_of_bounds or in_place or tma" 2>&1 | tail -2
for b in 8 64 256 1024; do for t in 1 0; do echo "bpr=$b TMA=$t"; GAES_ROWS_TMA=$t python scripts/profile_kernels.py cbc_rows 24 $b; done; done
for t in 1 0; do GAES_ROWS_TMA=$t python scripts/profile_kernels.py cbc_rows 20 64; GAES_ROWS_TMA=$t python scripts/profile_kernels.py cbc_rows 20 256; done
