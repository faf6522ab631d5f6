#!/bin/bash
# round-2 GPU batch L: ncu source profile of the tensor-core wide kernel
set -x
O=gpurun_out/r2l; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modexp_tcw -s 1 -c 1 -o $O/ncu_tcw_full python tools/tcw_one.py 3072 3072 37888 > $O/ncu_tcw_full.log 2>&1
ls -la $O
