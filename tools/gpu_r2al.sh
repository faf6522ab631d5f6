#!/bin/bash
# round-2 GPU batch AL: k = 33 modexp kernel with 3 tiles (own 144-column accumulators, up to 168 registers, t3.so) vs 4
# tiles sharing 3 slots (t4.so): C2 / C5 A/B, parity of t3 on the tensor paths
set -x
O=gpurun_out/r2al; mkdir -p $O
bash tools/gpu_ab_c2.sh t4.so t3.so > /dev/null 2>&1
cp gpurun_out/ab_c2/ab.log $O/ab.log
MR_RNS_LIB=$PWD/tools/ab/t3.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py -x -q > $O/pytest_t3.log 2>&1; echo "pytest exit $?" >> $O/pytest_t3.log
cat $O/ab.log
