timeout 1200 python -m pytest tests/test_gpu_mr.py -x -q -k "wide_candidates" > gpurun_out/pytest_mrw.log 2>&1; echo "exit $?" >> gpurun_out/pytest_mrw.log
