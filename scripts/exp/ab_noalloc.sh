# Input loads: texture path (default) vs LDG.cs vs LDG with L1::no_allocate
cp paper_1506_08503_b200/libgaes_b200.so /tmp/base.so
for r in 1 2; do
  echo -n "tex (base): "; python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])['value'])"
  echo -n "ldg.cs (base, GAES_TEXIN=0): "; GAES_TEXIN=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])['value'])"
  cp scripts/exp/alt/libgaes_b200.so paper_1506_08503_b200/libgaes_b200.so
  echo -n "ldg.no_allocate (alt, GAES_TEXIN=0): "; GAES_TEXIN=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])['value'])"
  cp /tmp/base.so paper_1506_08503_b200/libgaes_b200.so
done
