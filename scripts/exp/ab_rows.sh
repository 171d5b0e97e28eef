cp paper_1506_08503_b200/libgaes_b200.so /tmp/base.so
for round in 1 2; do
  for v in base alt; do
    if [ $v = base ]; then cp /tmp/base.so paper_1506_08503_b200/libgaes_b200.so; else cp scripts/exp/alt/libgaes_b200.so paper_1506_08503_b200/libgaes_b200.so; fi
    echo -n "$v "; python scripts/profile_kernels.py cbc_dec_rows 24 64; echo -n "$v "; python scripts/profile_kernels.py cbc_dec_rows 24 4
  done
done
cp /tmp/base.so paper_1506_08503_b200/libgaes_b200.so
