#!/bin/bash
# round-2 GPU batch H: first run of the tensor-core wide kernel (k = 97 / 129)
set -x
O=gpurun_out/r2h; mkdir -p $O
timeout 300 python tools/tcw_probe.py > $O/probe.log 2>&1; echo "exit $?" >> $O/probe.log
#MR_RNS_TCW=0 timeout 300 python tools/tcw_probe.py > $O/probe_imad.log 2>&1; echo "exit $?" >> $O/probe_imad.log
ls -la $O
