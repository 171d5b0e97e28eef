set -e
python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python scripts/exp/small_probe.py | head -3
python bench.py --config 1 --no-cpu-baseline > gpurun_out/b1.json
python bench.py --no-cpu-baseline > gpurun_out/b2.json
python -c "
import json
for c in (1, 2):
    d = json.load(open(f'gpurun_out/b{c}.json')); print(c, d['value'], d['ms_per_step'], d['decrypt_gbs_per_gpu'], d['e2e']['value'])"
