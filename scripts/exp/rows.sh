for t in 1 0 1 0; do
GAES_TEXIN=$t python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b2.json; python -c "
import json; d=json.load(open('gpurun_out/b2.json')); print('TEXIN=$t', d['value'], d['decrypt_gbs_per_gpu'])"
done
