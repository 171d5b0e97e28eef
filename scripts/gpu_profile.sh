#!/usr/bin/env bash
# Run on the GPU box (via gpurun): plain bench, the ncu launch list and one
# `ncu --set full` capture of the dominant kernel.  Usage:
#   scripts/gpu_profile.sh <tag> [bench args...]
set -uo pipefail
TAG="${1:-r1}"; shift || true
ARGS="${*:---config 2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e}"
OUT=gpurun_out
mkdir -p "$OUT"
CMD="python bench.py $ARGS"
$CMD > "$OUT/${TAG}_plain.json" 2> "$OUT/${TAG}_plain.err" || { echo "plain run failed"; tail -20 "$OUT/${TAG}_plain.err"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/${TAG}_launches.csv" $CMD > "$OUT/${TAG}_ncu_launches.log" 2>&1 || echo "launch list failed"
ncu --set full --clock-control none --import-source on -k regex:k_blocks -s 4 -c 1 \
    -o "$OUT/${TAG}_prof" $CMD > "$OUT/${TAG}_ncu_full.log" 2>&1 || echo "ncu full failed"
ls -la "$OUT"
