#!/bin/bash
# round-2 GPU batch O: tensor-core wide kernel at k = 257 (8192-bit moduli, 16,128-bit CRT keys): parity tests, W configs,
# ncu of the k = 257 kernel
set -x
O=gpurun_out/r2o; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_tcw.py -x -q > $O/pytest_tcw.log 2>&1; echo "pytest exit $?" >> $O/pytest_tcw.log
timeout 900 python tools/bench_configs.py --configs W > $O/configs_w.jsonl 2> $O/configs_w.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modexp_tcw -s 1 -c 1 -o $O/ncu_tcw257_enc python tools/tcw_one.py 8192 17 18944 > $O/ncu_tcw257_enc.log 2>&1
ls -la $O
