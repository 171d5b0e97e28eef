# A/B of the general-M CBC encrypt row kernels: in-tree .so (base) vs
# scripts/exp/alt/libgaes_b200.so (alt), two rounds, several row lengths.
cp paper_1506_08503_b200/libgaes_b200.so /tmp/base.so
for round in 1 2; do
  for v in base alt; do
    if [ $v = base ]; then cp /tmp/base.so paper_1506_08503_b200/libgaes_b200.so; else cp scripts/exp/alt/libgaes_b200.so paper_1506_08503_b200/libgaes_b200.so; fi
    for shape in "24 8" "24 64" "24 128" "26 64"; do echo -n "$v $shape: "; python scripts/profile_kernels.py cbc_rows $shape; done
  done
done
cp scripts/exp/alt/libgaes_b200.so paper_1506_08503_b200/libgaes_b200.so
python scripts/exp/tma_rows_probe.py
cp /tmp/base.so paper_1506_08503_b200/libgaes_b200.so
