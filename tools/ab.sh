#!/bin/bash
# usage: bash tools/ab.sh libA.so libB.so ...  — alternate bench runs per library (in tools/ab/), ladder ms
for rep in 1 2; do
  for lib in "$@"; do
    MR_RNS_LIB=$PWD/tools/ab/$lib python bench.py --no-cpu-baseline --no-verify 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$lib', round(d['value']), round(r['frac'],4), round(r['ladder_ms_per_launch'],3))"
  done
done
