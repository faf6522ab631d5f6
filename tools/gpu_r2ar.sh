#!/bin/bash
# round-2 GPU batch AR: top-down exit comparison in the thread-per-message exit (from_rns) and the lanes kernel's exit
# (cmptop.so) vs before.so: parity (paths, parity, Miller-Rabin), C1 probe, C4 / C2 A/B
set -x
O=gpurun_out/r2ar; mkdir -p $O
MR_RNS_LIB=$PWD/tools/ab/cmptop.so timeout 1800 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_mr.py -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
for rep in 1 2; do
  for lib in cmptop before; do
    echo "== $lib" >> $O/ab.log
    MR_RNS_LIB=$PWD/tools/ab/$lib.so timeout 300 python tools/c1_probe.py >> $O/ab.log 2>&1
    MR_RNS_LIB=$PWD/tools/ab/$lib.so timeout 600 python tools/bench_configs.py --configs C4 2>/dev/null | head -2 | cut -c1-120 >> $O/ab.log
    MR_RNS_LIB=$PWD/tools/ab/$lib.so timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-verify 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c2', round(d['value']))" >> $O/ab.log
  done
done
cat $O/ab.log
