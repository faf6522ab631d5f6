#!/bin/bash
# usage: bash tools/gpu_check.sh TAG [full]   — GPU tests (both kernel paths), bench, ncu launch list (+ full ncu)
TAG=${1:-x}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15
MR_RNS_IMAD_ONLY=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
MR_RNS_IMAD_ONLY=1 python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}_imad.json 2>&1; cat gpurun_out/bench_${TAG}_imad.json | head -c 600; echo
if [ "$2" == "full" ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-verify --no-cpu-baseline > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_modexp -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-verify --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
  tail -2 gpurun_out/ncu_$TAG.log
fi
