#!/bin/bash
# round-2 GPU batch R: k = 33 with all 33 outputs on the tensor core and 4 tiles sharing 3 TMEM accumulator slots
# (tools/ab/nt33s.so) vs 3 tiles (nt33.so) vs the default (frac.so: 32 outputs + 1 CUDA-core column): parity of
# nt33s on the k = 33 tensor paths, then C2/C5 A/B
set -x
O=gpurun_out/r2r; mkdir -p $O
MR_RNS_LIB=$PWD/tools/ab/nt33s.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py -x -q > $O/pytest_nt33s.log 2>&1; echo "pytest exit $?" >> $O/pytest_nt33s.log
bash tools/gpu_ab_c2.sh frac.so nt33s.so nt33.so > /dev/null 2>&1
cp gpurun_out/ab_c2/ab.log $O/ab.log
cat $O/ab.log
