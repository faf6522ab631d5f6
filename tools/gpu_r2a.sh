#!/bin/bash
# round-2 GPU batch A: tests, peak microbenchmarks, sanitizer logs, bench (run under gpurun)
set -x
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2a/build.log 2>&1
(cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o n9_intpeak n9_intpeak.cu && ./n9_intpeak) > gpurun_out/r2a/n9_intpeak.jsonl 2>&1
(cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tc_i8_peak tc_i8_peak.cu && timeout 120 ./tc_i8_peak) > gpurun_out/r2a/tc_i8_peak.jsonl 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2a/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2a/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err
for c in crt33 pair65 mr33 wide97 imad33 drbg keygen; do
  timeout 900 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize_smoke.py $c > gpurun_out/r2a/san_memcheck_$c.log 2>&1
  echo "exit $?" >> gpurun_out/r2a/san_memcheck_$c.log
done
for t in racecheck synccheck; do
  for c in crt33 pair65 mr33 wide97 imad33; do
    timeout 900 compute-sanitizer --tool $t python tools/sanitize_smoke.py $c > gpurun_out/r2a/san_${t}_$c.log 2>&1
    echo "exit $?" >> gpurun_out/r2a/san_${t}_$c.log
  done
done
ls -la gpurun_out/r2a
