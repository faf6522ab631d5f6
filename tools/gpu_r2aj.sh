#!/bin/bash
# round-2 GPU batch AI: lanes kernel also keeps its per-channel / per-output constants in registers (lpo8.so vs creg.so):
# small-batch parity, C1 A/B vs MR_LANES_CREG=0
set -x
O=gpurun_out/r2aj; mkdir -p $O
MR_RNS_LIB=$PWD/tools/ab/lpo8.so timeout 1500 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
for rep in 1 2; do
  for lib in lpo8 lpo4; do
    echo "== $lib" >> $O/ab.log
    MR_RNS_LIB=$PWD/tools/ab/$lib.so timeout 300 python tools/c1_probe.py >> $O/ab.log 2>&1
  done
done
cat $O/ab.log
