#!/bin/bash
# round-2 GPU batch I: tcw parity tests, full GPU suite, ncu of the tensor-core wide kernel
set -x
O=gpurun_out/r2i; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tcw.py -x -q > $O/pytest_tcw.log 2>&1; echo "exit $?" >> $O/pytest_tcw.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modexp_tcw -s 1 -c 1 -o $O/ncu_tcw_enc python tools/tcw_one.py 3072 17 65536 > $O/ncu_tcw_enc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modexp_tcw -s 1 -c 1 -o $O/ncu_tcw_full python tools/tcw_one.py 3072 3072 4096 > $O/ncu_tcw_full.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
ls -la $O
