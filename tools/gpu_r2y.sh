#!/bin/bash
# round-2 GPU batch Y: small-batch threshold sweep (MR_RNS_SMALL_MAX = jobs x contexts at or below which the lanes kernel
# runs): C1 and the C3 sizes 1K / 4K / 16K
O=gpurun_out/r2y; mkdir -p $O; : > $O/sweep.jsonl
for sm in 0 1024 2048 4096 8192; do
  MR_RNS_SMALL_MAX=$sm timeout 600 python tools/bench_configs.py --configs C1,C3 --quick 2>/dev/null | sed "s/^{/{\"small_max\": $sm, /" >> $O/sweep.jsonl
done
cut -c1-200 $O/sweep.jsonl
