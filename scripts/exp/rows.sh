for t in 1 2 1 2; do
GAES_ILP=$t python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b2.json; python -c "
import json; d=json.load(open('gpurun_out/b2.json')); print('ILP=$t', d['value'], d['decrypt_gbs_per_gpu'])"
GAES_ILP=$t python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/b3.json; python -c "
import json; d=json.load(open('gpurun_out/b3.json')); print('ILP=$t cfg3', d['value'], d['decrypt_gbs_per_gpu'])"
done
