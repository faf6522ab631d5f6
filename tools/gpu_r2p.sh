#!/bin/bash
# round-2 GPU batch P: CTA-pair streaming (MR_TCW_PAIR=1, tools/ab/pair.so) vs the single-CTA tensor-core wide kernel:
# parity of the pair build on the tcw tests, then the tcw probe A/B (both builds, twice)
set -x
O=gpurun_out/r2p; mkdir -p $O
MR_RNS_LIB=$PWD/tools/ab/pair.so timeout 600 python tools/tcw_probe.py quick > $O/pair_quick.log 2>&1; echo "exit $?" >> $O/pair_quick.log
MR_RNS_LIB=$PWD/tools/ab/pair.so timeout 1500 python -m pytest tests/test_gpu_tcw.py -x -q > $O/pytest_tcw_pair.log 2>&1; echo "pytest exit $?" >> $O/pytest_tcw_pair.log
cp paper_1305_3699_b200/libmr_rns.so tools/ab/base.so
for rep in 1 2; do
  for lib in base pair; do
    echo "== $lib rep $rep" >> $O/ab.log
    MR_RNS_LIB=$PWD/tools/ab/$lib.so timeout 300 python tools/tcw_probe.py 2>&1 | grep throughput >> $O/ab.log
  done
done
cat $O/ab.log
