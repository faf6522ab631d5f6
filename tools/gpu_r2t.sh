#!/bin/bash
# round-2 GPU batch T: accumulator slots freed per warp (MR_TC_RELWARP=1, relwarp.so) vs a tile barrier (base.so = r2s):
# parity of relwarp on the k <= 65 tensor paths, C2 / C5 A/B
set -x
O=gpurun_out/r2t; mkdir -p $O
MR_RNS_LIB=$PWD/tools/ab/relwarp.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py tests/test_gpu_mr.py -x -q > $O/pytest_relwarp.log 2>&1; echo "pytest exit $?" >> $O/pytest_relwarp.log
bash tools/gpu_ab_c2.sh base.so relwarp.so > /dev/null 2>&1
cp gpurun_out/ab_c2/ab.log $O/ab.log
cat $O/ab.log
