#!/bin/bash
# round-2 GPU batch V: tensor-core wide kernel at k = 505 (64-message tiles, M = 64, B residues in global scratch):
# quick parity probe (all tcw k), the tcw GPU tests, W configs, ncu of the k = 505 kernel
set -x
O=gpurun_out/r2v; mkdir -p $O
timeout 600 python tools/tcw_probe.py quick > $O/probe_quick.log 2>&1; echo "exit $?" >> $O/probe_quick.log
timeout 1800 python -m pytest tests/test_gpu_tcw.py -x -q > $O/pytest_tcw.log 2>&1; echo "pytest exit $?" >> $O/pytest_tcw.log
timeout 900 python tools/bench_configs.py --configs W > $O/configs_w.jsonl 2> $O/configs_w.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modexp_tcw -s 1 -c 1 -o $O/ncu_tcw505_enc python tools/tcw_one.py 16128 17 9472 > $O/ncu_tcw505.log 2>&1
ls -la $O
