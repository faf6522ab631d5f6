#!/bin/bash
# round-2 GPU batch U: C1 small-batch profile (ncu of the k_modexp_lane launch of the full-d decryption) and the C3 sweep
# to 1M messages
set -x
O=gpurun_out/r2u; mkdir -p $O
timeout 300 python tools/c1_probe.py > $O/c1_probe.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modexp_lane -s 3 -c 1 -o $O/ncu_c1_fulld python tools/c1_probe.py 1 > $O/ncu_c1.log 2>&1
timeout 900 python tools/bench_configs.py --configs C3 > $O/configs_c3.jsonl 2> $O/configs_c3.err
ls -la $O
