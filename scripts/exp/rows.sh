python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python bench.py --no-cpu-baseline > gpurun_out/b2.json; python -c "
import json; d=json.load(open('gpurun_out/b2.json')); print(d['value'], d['e2e']['value'], d['e2e_dropin']['value'], d['roofline']['frac'], d['gpu_launches'])"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
