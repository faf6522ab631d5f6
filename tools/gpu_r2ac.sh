#!/bin/bash
# round-2 GPU batch AC: compute-sanitizer memcheck / racecheck / synccheck of the session-3 kernels (k = 33 tensor kernel
# with shared accumulator slots via crt33, the tensor-core wide kernel at k = 97 / 257 / 505, the lanes kernel), then the
# Miller-Rabin N = 144 A/B (mrnt33.so vs final.so) on C5
O=gpurun_out/r2ac; mkdir -p $O
for c in crt33 wide97 tcw257 tcw505 lanes33; do
  timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_smoke.py $c > $O/san_memcheck_$c.log 2>&1
  for t in racecheck synccheck; do
    timeout 1200 compute-sanitizer --tool $t python tools/sanitize_smoke.py $c > $O/san_${t}_$c.log 2>&1
  done
done
for f in $O/san_*.log; do echo "$f: $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY\|sanitize_smoke' $f | tr '\n' ' ')"; done > $O/summary.txt
for rep in 1 2; do
  for lib in final.so mrnt33.so; do
    MR_RNS_LIB=$PWD/tools/ab/$lib timeout 300 python bench.py --workload c5 --steps 5 --no-cpu-baseline --no-verify 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'c5', round(d['value']))" >> $O/ab_mr.log
  done
done
cat $O/summary.txt $O/ab_mr.log
