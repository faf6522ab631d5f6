#!/bin/bash
# round-2 GPU batch AG: ncu of the C1 full-d decryption on the lanes kernel (after the fractional α')
O=gpurun_out/r2ag; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modexp_lane -s 3 -c 1 -o $O/ncu_c1_fulld python tools/c1_probe.py 1 > $O/ncu_c1.log 2>&1
ls -la $O
