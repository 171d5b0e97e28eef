python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python scripts/exp/small_graph_probe.py
./scripts/exp/launch_probe | grep graph
for i in 1 2; do
python bench.py --config 1 --no-cpu-baseline --no-e2e > gpurun_out/b1.json; python -c "
import json; d=json.load(open('gpurun_out/b1.json')); print('cfg1', d['value'], d['decrypt_gbs_per_gpu'])"
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b2.json; python -c "
import json; d=json.load(open('gpurun_out/b2.json')); print('cfg2', d['value'], d['decrypt_gbs_per_gpu'])"
done
