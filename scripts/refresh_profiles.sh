#!/usr/bin/env bash
# Run on the GPU box (via gpurun): the GPU test suite, the default bench line,
# every config's bench line, the reference arm, the ncu launch list of the
# default bench and one `ncu --set full` capture of the headline kernel.
# Everything lands in gpurun_out/final/ (copied into profiles/ afterwards).
set -uo pipefail
OUT=gpurun_out/final
mkdir -p "$OUT"
python -m pytest tests -q -m gpu > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" | tee -a "$OUT/status.txt"
tail -3 "$OUT/pytest_gpu.log"
python bench.py > "$OUT/bench_default.json" 2> "$OUT/bench_default.err"; echo "bench rc=$?" | tee -a "$OUT/status.txt"
for c in 1 2 3 4 5; do
  python bench.py --config $c > "$OUT/bench_cfg$c.json" 2> "$OUT/bench_cfg$c.err"; echo "cfg$c rc=$?" | tee -a "$OUT/status.txt"
done
python bench.py --impl reference > "$OUT/bench_reference_arm.json" 2> "$OUT/bench_reference_arm.err"; echo "ref rc=$?" | tee -a "$OUT/status.txt"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" $CMD > "$OUT/ncu_launches.log" 2>&1; echo "ncu launches rc=$?" | tee -a "$OUT/status.txt"
ncu --set full --clock-control none --import-source on -k regex:k_blocks -s 4 -c 1 -o "$OUT/ttable_prof" $CMD > "$OUT/ncu_full.log" 2>&1; echo "ncu full rc=$?" | tee -a "$OUT/status.txt"
ls -la "$OUT"
