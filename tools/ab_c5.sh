#!/bin/bash
# usage: bash tools/ab_c5.sh libA.so libB.so ...  — C5 (Miller-Rabin) per library (in tools/ab/)
for rep in 1 2; do
  for lib in "$@"; do
    MR_RNS_LIB=$PWD/tools/ab/$lib python tools/bench_configs.py --configs C5 2>/dev/null | grep '"C5"' | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$lib', round(d['forced_rounds_per_s']), round(d['early_exit_candidates_per_s']), d['bit_exact_sample_vs_oracle'], d['verdicts_equal_forced_vs_early_exit'])"
  done
done
