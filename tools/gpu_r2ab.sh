#!/bin/bash
# round-2 GPU batch AB: whole GPU suite on the final session-3 build (tcw fractional α'), twice the multi-job tcw test,
# smoke(), default bench
set -x
O=gpurun_out/r2ab; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_tcw.py -q -k several_jobs >> $O/multijob.log 2>&1; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 300 python bench.py > $O/bench.json 2> $O/bench.err
ls -la $O
