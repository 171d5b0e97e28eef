mkdir -p gpurun_out/traffic
for c in 1 3 4 5; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
      -k regex:"k_blocks|k_many_key" -s 4 -c 1 \
      python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/traffic/cfg$c.csv 2> gpurun_out/traffic/cfg$c.err
  echo cfg$c rc=$?
done
