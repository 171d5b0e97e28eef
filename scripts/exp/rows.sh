python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python bench.py --no-cpu-baseline > gpurun_out/b2.json; python -c "
import json; d=json.load(open('gpurun_out/b2.json')); print(d['value'], d['decrypt_gbs_per_gpu'], d['e2e']['value']); print(json.dumps(d['roofline'], indent=1))"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:k_blocks -s 4 -c 1 -o gpurun_out/texs_prof $CMD > gpurun_out/texs_ncu.log 2>&1; echo ncu rc=$?
