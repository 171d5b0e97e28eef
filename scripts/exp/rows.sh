set -e
python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python scripts/exp/dropin_probe.py
python bench.py > gpurun_out/b2.json; python -c "
import json; d=json.load(open('gpurun_out/b2.json')); print('cfg2', d['value'], d['e2e']['value'], d.get('e2e_dropin'))"
