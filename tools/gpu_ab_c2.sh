#!/bin/bash
# A/B of builds (tools/ab/*.so) on C2 (bench.py defaults) and C5, twice, alternating
O=gpurun_out/ab_c2; mkdir -p $O; : > $O/ab.log
for rep in 1 2; do
  for lib in "$@"; do
    for wl in c2 c5; do
      MR_RNS_LIB=$PWD/tools/ab/$lib timeout 300 python bench.py --workload $wl --steps 5 --no-cpu-baseline --no-verify 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$wl', round(d['value']), round(d['roofline']['ladder_ms_per_launch'],3))" >> $O/ab.log
    done
  done
done
cat $O/ab.log
