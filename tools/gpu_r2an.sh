#!/bin/bash
# round-2 GPU batch AN: sliding-window cap A/B on C2 (MR_RNS_WMAX = 7 (default), 6, 5, 4)
O=gpurun_out/r2an; mkdir -p $O; : > $O/ab.log
for rep in 1 2; do
  for w in 7 6 5 4; do
    MR_RNS_WMAX=$w timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-verify 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('wmax $w', round(d['value']), round(d['roofline']['ladder_ms_per_launch'],3))" >> $O/ab.log
  done
done
cat $O/ab.log
