python -m pytest tests -x -q -m gpu -k "cbc or grid or iv or aliased or in_place or dropin_mixed" 2>&1 | tail -2
for i in 1 2; do
python scripts/profile_kernels.py cbc_dec_rows 24 64
python scripts/profile_kernels.py cbc_dec_rows 24 1
python scripts/profile_kernels.py cbc_dec_rows 24 4
done
