#!/usr/bin/env bash
# Round-2 end-of-round evidence on one B200 (via gpurun): GPU tests, smoke, the
# default bench line (config 3) and the reference arm, every config's line, the
# launch list + one `ncu --set full` capture of the dominant kernel for the
# default command, captures of the new kernels, DRAM traffic per config,
# sweeps.  Output: gpurun_out/r2final/ (summaries are copied into profiles/r2/).
set -uo pipefail
O=gpurun_out/r2final; mkdir -p $O
st() { echo "$1 rc=$2" | tee -a $O/status.txt; }
timeout 1800 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; st pytest $?
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; st smoke $?
python bench.py > $O/bench_default.json 2> $O/bench_default.err; st bench $?
for r in 2 3; do python bench.py --no-cpu-baseline > $O/bench_default_rep$r.json 2> $O/bench_default_rep$r.err; st bench_rep$r $?; done
python bench.py --impl reference > $O/bench_reference_arm.json 2> $O/bench_reference_arm.err; st ref $?
for c in 1 2 4 5; do
  python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; st cfg$c $?
done
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > $O/plain_default.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_default.csv $CMD > $O/ncu_launches.log 2>&1; st ncu_launches $?
$CMD > $O/plain_default2.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_blocks -s 4 -c 1 -o $O/ttable_cfg3 $CMD > $O/ncu_full.log 2>&1; st ncu_full $?
CMD1="python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD1 > $O/plain_cfg1.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_cfg1.csv $CMD1 > $O/ncu_launches1.log 2>&1; st ncu_launches_cfg1 $?
$CMD1 > $O/plain_cfg1b.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_blocks_small -s 12 -c 1 -o $O/small_cfg1 $CMD1 > $O/ncu_small.log 2>&1; st ncu_small $?
python scripts/profile_kernels.py cbc_rows 20 4096 > $O/plain_quad.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_cbc_enc_rows_quad -s 2 -c 1 -o $O/rows_quad python scripts/profile_kernels.py cbc_rows 20 4096 > $O/ncu_quad.log 2>&1; st ncu_quad $?
for c in 3 4 5; do
  python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/plain_t$c.json 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
      -k regex:"k_blocks|k_many_key" -s 4 -c 1 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/traffic_cfg$c.csv 2> $O/traffic_cfg$c.err; st traffic$c $?
done
python -m paper_1506_08503_b200.sweep --kind count --counts 1,10,100,1000,10000,100000,1000000,16777216 --out $O/sweep_count_cuda.csv > $O/sweeps.log 2>&1; st sweep1 $?
python -m paper_1506_08503_b200.sweep --kind count --device-resident --counts 1024,16384,65536,262144,1048576,4194304,16777216,67108864,268435456 --out $O/sweep_count_cuda_device.csv >> $O/sweeps.log 2>&1; st sweep2 $?
python -m paper_1506_08503_b200.sweep --kind length --n-messages 100000 --lengths 16,64,256,1024,4096 --out $O/sweep_length_cuda.csv >> $O/sweeps.log 2>&1; st sweep3 $?
python -m paper_1506_08503_b200.sweep --kind length --device-resident --n-messages 262144 --lengths 16,32,64,256,1024,4096 --out $O/sweep_length_cuda_device.csv >> $O/sweeps.log 2>&1; st sweep4 $?
ls -la $O
