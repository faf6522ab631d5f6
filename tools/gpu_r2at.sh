#!/bin/bash
# round-2 GPU batch AT: last A/Bs — two compute warps per lane quadrant in the k = 97 / 129 wide kernel (halves2.so) and
# suspend-hinted MMA waits in the k <= 65 tensor kernels (waithint.so) vs the final build (base.so)
O=gpurun_out/r2at; mkdir -p $O; : > $O/ab.log
for rep in 1 2; do
  for lib in base halves2; do
    echo "== $lib" >> $O/ab.log
    MR_RNS_LIB=$PWD/tools/ab/$lib.so timeout 600 python tools/tcw_probe.py 2>&1 | grep "throughput bits=\(3072\|4096\)" >> $O/ab.log
  done
done
bash tools/gpu_ab_c2.sh base.so waithint.so > /dev/null 2>&1
cat gpurun_out/ab_c2/ab.log >> $O/ab.log
cat $O/ab.log
