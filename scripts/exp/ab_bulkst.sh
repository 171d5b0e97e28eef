# M = 16 encrypt: per-lane STG.128 (default) vs shared-memory tile + bulk copy (GAES_BULKST=1)
for r in 1 2 3; do
  for v in 0 1; do
    echo -n "GAES_BULKST=$v: "; GAES_BULKST=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['verified'])"
  done
done
for v in 0 1; do echo -n "cfg3 GAES_BULKST=$v: "; GAES_BULKST=$v python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['verified'])"; done
