#!/bin/bash
# usage: bash tools/ab_w.sh libA.so libB.so ...  — wide-operand configuration (W) per library (in tools/ab/)
for lib in "$@"; do
  MR_RNS_LIB=$PWD/tools/ab/$lib python tools/bench_configs.py --configs W 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$lib', d['modulus_bits'], d['exponent_bits'], round(d['modexps_per_s'],1), round(d['imad_eq_frac'],3), d['bit_exact_sample'])"
done
