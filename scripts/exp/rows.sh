for e in 0 2 0 2; do
echo "GAES_EARLY=$e"
GAES_EARLY=$e python scripts/exp/small_graph_probe.py 2>&1 | grep -E "2\^(14|16|18)"
GAES_EARLY=$e python bench.py --config 1 --no-cpu-baseline --no-e2e > gpurun_out/b1.json; python -c "
import json; d=json.load(open('gpurun_out/b1.json')); print('cfg1', d['value'], d['decrypt_gbs_per_gpu'])"
done
