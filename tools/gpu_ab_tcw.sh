#!/bin/bash
# A/B of tensor-core wide kernel builds (tools/ab/*.so): probe throughput per library, twice, alternating
O=gpurun_out/ab_tcw; mkdir -p $O
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib rep $rep" >> $O/ab.log
    MR_RNS_LIB=$PWD/tools/ab/$lib timeout 300 python tools/tcw_probe.py 2>&1 | grep -v "^bits" >> $O/ab.log
  done
done
cat $O/ab.log
