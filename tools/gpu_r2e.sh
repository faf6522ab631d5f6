#!/bin/bash
# round-2 GPU batch E: ncu of the small-batch kernel, A/B of the ALU byte-column combine
set -x
O=gpurun_out/r2e; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modexp_wide -s 1 -c 1 -o $O/ncu_lanes python tools/lanes_probe.py lanes > $O/ncu_lanes.log 2>&1
bash tools/ab.sh base.so alu.so > $O/ab_alu.txt 2>&1
ls -la $O
