timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for b in 8 16 32 64 128 256; do echo "bpr=$b"; python scripts/profile_kernels.py cbc_rows 24 $b; done
python scripts/profile_kernels.py cbc_rows 26 64
