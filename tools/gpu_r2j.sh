#!/bin/bash
# round-2 GPU batch J: two-tile tensor-core wide kernel: probe, tcw tests, ncu
set -x
O=gpurun_out/r2j; mkdir -p $O
timeout 300 python tools/tcw_probe.py > $O/probe.log 2>&1; echo "exit $?" >> $O/probe.log
timeout 900 python -m pytest tests/test_gpu_tcw.py -x -q > $O/pytest_tcw.log 2>&1; echo "exit $?" >> $O/pytest_tcw.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modexp_tcw -s 1 -c 1 -o $O/ncu_tcw_full python tools/tcw_one.py 3072 3072 37888 > $O/ncu_tcw_full.log 2>&1
ls -la $O
