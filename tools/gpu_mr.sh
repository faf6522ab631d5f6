#!/bin/bash
# MR tensor path: parity tests on both paths + C5 measurement
timeout 600 python -m pytest tests/test_gpu_mr.py -x -q -m gpu 2>&1 | tail -5
MR_RNS_IMAD_ONLY=1 timeout 600 python -m pytest tests/test_gpu_mr.py -x -q -m gpu 2>&1 | tail -2
python tools/bench_configs.py --configs C5 2>&1 | tee gpurun_out/c5_$1.jsonl
MR_RNS_IMAD_ONLY=1 python tools/bench_configs.py --configs C5 2>&1 | tee gpurun_out/c5_$1_imad.jsonl
