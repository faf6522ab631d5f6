#!/bin/bash
# usage: bash tools/ab_c3.sh libA.so ...  — C3 (RSA-3072) per library (in tools/ab/)
for lib in "$@"; do
  MR_RNS_LIB=$PWD/tools/ab/$lib python tools/bench_configs.py --configs C3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['encrypt_ops_per_s']), round(d['decrypt_crt_ops_per_s']), d['bit_exact'])"
done
