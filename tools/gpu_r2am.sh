#!/bin/bash
# round-2 GPU batch AM: GPU suite + smoke + default bench on the last commit of the round (per-device tcw attribute)
set -x
O=gpurun_out/r2am; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 300 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
ls -la $O
