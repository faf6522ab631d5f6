#!/bin/bash
# round-2 GPU batch D: small-batch kernel (mr_lanes.cu) parity on all paths + crossover sweep
set -x
O=gpurun_out/r2d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_paths.py -x -q > $O/pytest_paths.log 2>&1; echo "exit $?" >> $O/pytest_paths.log
timeout 900 python tools/small_sweep.py > $O/small_sweep.jsonl 2> $O/small_sweep.err
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
ls -la $O
