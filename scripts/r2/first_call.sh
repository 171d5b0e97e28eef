#!/usr/bin/env bash
# Round-2 first GPU call: small-batch decomposition, per-instruction bank
# conflicts of the headline kernel (texture paths on / off), config-3 bench line.
set -u
mkdir -p gpurun_out/r2a
O=gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python scripts/exp/small_probe.py > $O/small_probe.txt 2>&1
python scripts/exp/small_graph_probe.py > $O/small_graph_probe.txt 2>&1
python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python scripts/profile_kernels.py encrypt 24 > $O/plain_tex.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_blocks -s 3 -c 1 \
      -o $O/ttable_src python scripts/profile_kernels.py encrypt 24 > $O/ncu_tex.log 2>&1
GAES_TUNE=TEXS=0,TEXIN=0 python scripts/profile_kernels.py encrypt 24 > $O/plain_notex.log 2>&1 && \
  GAES_TUNE=TEXS=0,TEXIN=0 ncu --set full --clock-control none --import-source on -k regex:k_blocks -s 3 -c 1 \
      -o $O/ttable_notex_src python scripts/profile_kernels.py encrypt 24 > $O/ncu_notex.log 2>&1
ls -la $O
