set -e
python -m pytest tests -x -q -m gpu -k "probes or launch_counter" 2>&1 | tail -2
python bench.py --no-cpu-baseline > gpurun_out/b2.json
python -c "
import json
d = json.load(open('gpurun_out/b2.json')); print(json.dumps(d['roofline'], indent=1)); print(d['clocks'])"
