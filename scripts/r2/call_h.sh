#!/usr/bin/env bash
set -u
O=gpurun_out/r2h; mkdir -p $O
for pos in 0 1 2; do for lim in 1536 0; do
  GAES_TUNE=SMALL_PDL_POS=$pos,SMALL_BLOCKS_PER_SM=$lim python bench.py --config 1 --no-cpu-baseline --no-e2e > $O/cfg1_pos${pos}_lim${lim}.json 2>&1
  python -c "import json; d=json.loads(open('$O/cfg1_pos${pos}_lim${lim}.json').read().strip().splitlines()[-1]); print('pos=$pos lim=$lim', round(d['ms_per_step']*1e3,3), 'us', d['value'], 'stream', d['stream_launch_steps']['ms_per_step']*1e3, 'dec', d['decrypt_gbs_per_gpu'], d['verified'])" >> $O/summary.txt
done; done
