# TMA row kernel vs LDG/STG row kernel below the default 24-groups-per-SM
# threshold (GAES_TUNE=ROWS_TMA_MIN_GROUPS=0 forces the TMA kernel).
for shape in "24 256" "24 128" "24 64" "22 64" "23 128" "24 512" "24 1024"; do
  for mg in 24 0; do
    echo -n "min_groups=$mg $shape: "; GAES_TUNE=ROWS_TMA_MIN_GROUPS=$mg python scripts/profile_kernels.py cbc_rows $shape
  done
done
