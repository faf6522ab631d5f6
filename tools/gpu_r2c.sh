#!/bin/bash
# round-2 GPU batch C: MR (L1 sigma/c2) tests + C5 bench + full-size ncu of the forced MR kernel
set -x
O=gpurun_out/r2c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_mr.py -x -q > $O/pytest_mr.log 2>&1; echo "exit $?" >> $O/pytest_mr.log
timeout 600 python tools/bench_configs.py --configs C5 > $O/configs_c5.jsonl 2> $O/configs_c5.err
timeout 600 python bench.py --workload c5 --count 65536 --steps 3 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mr_rounds_tc -s 0 -c 1 -o $O/ncu_mr_full python tools/bench_configs.py --configs C5 > $O/ncu_mr.log 2>&1
ls -la $O
