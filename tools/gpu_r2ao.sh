#!/bin/bash
# round-2 GPU batch AO: Miller-Rabin fixed window A/B on C5 (tools/bench_configs.py C5, MR_BENCH_WINDOW = 4, 5, 6)
O=gpurun_out/r2ao; mkdir -p $O; : > $O/ab.jsonl
for rep in 1 2; do
  for w in 5 4 6; do
    MR_BENCH_WINDOW=$w timeout 600 python tools/bench_configs.py --configs C5 2>/dev/null | sed "s/^{/{\"window\": $w, /" >> $O/ab.jsonl
  done
done
cut -c1-160 $O/ab.jsonl
