#!/usr/bin/env bash
O=gpurun_out/r2l; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_rows_quad.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python scripts/r2/rows_quad_probe.py > $O/rows_quad.txt 2>&1
