#!/bin/bash
# round-2 GPU batch K: timeline trace of the tensor-core wide kernel
set -x
O=gpurun_out/r2k; mkdir -p $O
rm -f /tmp/tcw.trace
MR_TCW_TRACE=/tmp/tcw.trace timeout 300 python tools/tcw_one.py 3072 3072 37888 > $O/trace_run.log 2>&1
cp /tmp/tcw.trace $O/tcw_full.trace
rm -f /tmp/tcw.trace
MR_TCW_TRACE=/tmp/tcw.trace timeout 300 python tools/tcw_one.py 3072 17 65536 >> $O/trace_run.log 2>&1
cp /tmp/tcw.trace $O/tcw_enc.trace
timeout 300 python tools/tcw_probe.py > $O/probe.log 2>&1
ls -la $O
