#!/bin/bash
# round-2 GPU batch AQ: 16-byte row loads / stores and the top-down exit comparison in the tensor-core wide kernel (vec.so) vs neither
# (novec.so): tcw GPU tests on vec, probe A/B (parity + throughput of every tcw k)
set -x
O=gpurun_out/r2aq; mkdir -p $O
MR_RNS_LIB=$PWD/tools/ab/vec.so timeout 1800 python -m pytest tests/test_gpu_tcw.py -q > $O/pytest_tcw.log 2>&1; echo "pytest exit $?" >> $O/pytest_tcw.log
for rep in 1 2; do
  for lib in vec novec; do
    echo "== $lib rep $rep" >> $O/ab.log
    MR_RNS_LIB=$PWD/tools/ab/$lib.so timeout 600 python tools/tcw_probe.py 2>&1 | grep -v "^bits.*ok=True" >> $O/ab.log
  done
done
cat $O/ab.log
