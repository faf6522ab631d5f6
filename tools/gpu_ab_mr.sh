#!/bin/bash
# A/B of Miller-Rabin builds (tools/ab/*.so): bench.py --workload c5 per library, twice, alternating
O=gpurun_out/ab_mr; mkdir -p $O; : > $O/ab.log
for rep in 1 2; do
  for lib in "$@"; do
    MR_RNS_LIB=$PWD/tools/ab/$lib timeout 300 python bench.py --workload c5 --steps 5 --no-cpu-baseline --no-verify 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value']), round(d['roofline']['ladder_ms_per_launch'],2))" >> $O/ab.log
  done
done
cat $O/ab.log
