#!/bin/bash
# round-2 GPU batch AS: final evidence of round 2 (last build: top-down exit comparison, 16-byte tcw rows)
# for 4 tiles, Miller-Rabin kernel unchanged (N = 128): full GPU tests, bench C2 / C5 / C3 enc, configs, launch list,
# ncu of the C2 kernel
set -x
O=gpurun_out/r2as; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --workload c5 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 300 python bench.py --workload c3enc > $O/bench_c3enc.json 2> $O/bench_c3enc.err
timeout 300 python bench.py --workload c3dec > $O/bench_c3dec.json 2> $O/bench_c3dec.err
timeout 1500 python tools/bench_configs.py --configs C1,C3,C4,C5,W > $O/configs.jsonl 2> $O/configs.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-verify --no-identity --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modexp -s 3 -c 1 -o $O/ncu_c2 python bench.py --steps 1 --warmup 3 --no-verify --no-identity --no-cpu-baseline > $O/ncu_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mr_rounds -s 1 -c 1 -o $O/ncu_mr python bench.py --workload c5 --steps 1 --warmup 1 --no-verify --no-identity --no-cpu-baseline > $O/ncu_mr.log 2>&1
ls -la $O
