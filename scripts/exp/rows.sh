python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for i in 1 2; do python scripts/profile_kernels.py rowiv_enc 24; python scripts/profile_kernels.py rowiv_dec 24; done
python scripts/profile_kernels.py cbc_dec_rows 24 64
