#!/usr/bin/env bash
O=gpurun_out/r2n; mkdir -p $O
(lscpu; nvidia-smi topo -m) > $O/topo.txt 2>&1
python scripts/r2/numa_probe.py > $O/numa.txt 2>&1
python scripts/r2/numa_probe.py >> $O/numa.txt 2>&1
