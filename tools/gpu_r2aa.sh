#!/bin/bash
# round-2 GPU batch AA: fractional α' in the tensor-core wide kernel (MR_TCW_FRAC=1, tcwfrac.so) vs the m_r channel
# (tcwnofrac.so): tcw GPU tests on the new build, probe A/B (parity + throughput, every tcw k)
set -x
O=gpurun_out/r2aa; mkdir -p $O
MR_RNS_LIB=$PWD/tools/ab/tcwfrac.so timeout 1800 python -m pytest tests/test_gpu_tcw.py -q > $O/pytest_tcw.log 2>&1; echo "pytest exit $?" >> $O/pytest_tcw.log
for rep in 1 2; do
  for lib in tcwfrac tcwnofrac; do
    echo "== $lib rep $rep" >> $O/ab.log
    MR_RNS_LIB=$PWD/tools/ab/$lib.so timeout 600 python tools/tcw_probe.py 2>&1 | grep -v "^bits.*ok=True" >> $O/ab.log
  done
done
cat $O/ab.log
