#!/bin/bash
# round-2 GPU batch AE: scaled BE1 epilogue without the fold of V (MR_EPI_NOFOLD=1, nofold.so): parity of the k <= 65
# tensor paths, C2 / C5 A/B vs fold.so
set -x
O=gpurun_out/r2ae; mkdir -p $O
MR_RNS_LIB=$PWD/tools/ab/nofold.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py tests/test_gpu_paths.py -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
bash tools/gpu_ab_c2.sh nofold.so fold.so > /dev/null 2>&1
cp gpurun_out/ab_c2/ab.log $O/ab.log
cat $O/ab.log
