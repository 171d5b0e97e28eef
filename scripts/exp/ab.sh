# A/B: the package library vs scripts/exp/alt/libgaes_b200.so (same sources, one define)
set -e
cp paper_1506_08503_b200/libgaes_b200.so /tmp/base.so
for round in 1 2; do
  for v in base alt; do
    if [ $v = base ]; then cp /tmp/base.so paper_1506_08503_b200/libgaes_b200.so; else cp scripts/exp/alt/libgaes_b200.so paper_1506_08503_b200/libgaes_b200.so; fi
    python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.json
    python -c "
import json; d = json.load(open('gpurun_out/ab_$v.json')); r = d['roofline']
print('$v', d['value'], 'dec', d['decrypt_gbs_per_gpu'], 'probe', r['probe_round_rate'], 'lds', r['peak'], d['clocks']['sm_mhz'])"
  done
done
cp /tmp/base.so paper_1506_08503_b200/libgaes_b200.so
