#!/usr/bin/env bash
# Run on the GPU box: plain timing + one `ncu --set full` capture per
# non-headline kernel (scripts/profile_kernels.py, 2^24 blocks).
set -uo pipefail
OUT=gpurun_out/kern
mkdir -p "$OUT"
run() {  # tag op regex [bpr]
  python scripts/profile_kernels.py "$2" 24 ${4:-64} > "$OUT/$1_plain.txt" 2>&1 || { echo "$1 plain failed"; return; }
  cat "$OUT/$1_plain.txt"
  ncu --set full --clock-control none --import-source on -k "regex:$3" -s 3 -c 1 -o "$OUT/$1_prof" \
      python scripts/profile_kernels.py "$2" 24 ${4:-64} > "$OUT/$1_ncu.log" 2>&1 || echo "$1 ncu failed"
}
run r1_decrypt decrypt "k_blocks"
run r1_manykey manykey "k_many_key"
run r1_cbc_rows cbc_rows "k_cbc_enc_rows" 64
run r1_cbc_dec_rows cbc_dec_rows "k_blocks" 64
run r1_rowiv_enc rowiv_enc "k_blocks"
ls "$OUT"
