#!/bin/bash
# round-2 GPU batch F: dedicated small-batch kernel (mr_lanes.cu k_modexp_lane) parity + crossover sweep
set -x
O=gpurun_out/r2f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_paths.py -x -q > $O/pytest_paths.log 2>&1; echo "exit $?" >> $O/pytest_paths.log
timeout 900 python tools/small_sweep.py > $O/small_sweep.jsonl 2> $O/small_sweep.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modexp_lane -s 1 -c 1 -o $O/ncu_lane python tools/lanes_probe.py lanes > $O/ncu_lane.log 2>&1
ls -la $O
