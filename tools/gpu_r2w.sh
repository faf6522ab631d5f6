#!/bin/bash
# round-2 GPU batch W: k = 505 tensor-core wide kernel after the table-load fix: probe (parity + throughput of every tcw
# k), the tcw GPU tests, W configs, ncu of the k = 505 kernel
set -x
O=gpurun_out/r2w; mkdir -p $O
timeout 900 python tools/tcw_probe.py > $O/probe.log 2>&1; echo "exit $?" >> $O/probe.log
timeout 1800 python -m pytest tests/test_gpu_tcw.py -q > $O/pytest_tcw.log 2>&1; echo "pytest exit $?" >> $O/pytest_tcw.log
timeout 900 python tools/bench_configs.py --configs W > $O/configs_w.jsonl 2> $O/configs_w.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modexp_tcw -s 1 -c 1 -o $O/ncu_tcw505_enc python tools/tcw_one.py 16128 17 9472 > $O/ncu_tcw505.log 2>&1
ls -la $O
