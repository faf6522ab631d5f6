#!/bin/bash
# round-2 GPU batch Q: fractional α' in the tensor kernels (MR_FRAC_ALPHA=1, no m_r upkeep): GPU parity of the default
# build on the k <= 65 tensor paths + Miller-Rabin, then A/B vs MR_FRAC_ALPHA=0 on C2 and C5
set -x
O=gpurun_out/r2q; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mr.py tests/test_gpu_concurrency.py -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
bash tools/gpu_ab_c2.sh frac.so nofrac.so > /dev/null 2>&1
cp gpurun_out/ab_c2/ab.log $O/ab.log
cat $O/ab.log
