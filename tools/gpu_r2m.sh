#!/bin/bash
# round-2 GPU batch M: tcw evidence — bench C3 encryption (tcw), ncu of the tcw kernel (full exponent and e = 65537),
# configs C3 + W
set -x
O=gpurun_out/r2m; mkdir -p $O
timeout 300 python bench.py --workload c3enc > $O/bench_c3enc.json 2> $O/bench_c3enc.err
MR_RNS_TCW=0 timeout 300 python bench.py --workload c3enc --no-cpu-baseline > $O/bench_c3enc_imadwide.json 2>&1
timeout 900 python tools/bench_configs.py --configs C3,W > $O/configs.jsonl 2> $O/configs.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modexp_tcw -s 1 -c 1 -o $O/ncu_tcw_full python tools/tcw_one.py 3072 3072 37888 > $O/ncu_tcw_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modexp_tcw -s 1 -c 1 -o $O/ncu_tcw_enc python tools/tcw_one.py 3072 17 65536 > $O/ncu_tcw_enc.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3enc.csv python bench.py --workload c3enc --steps 2 --warmup 3 --no-verify --no-identity --no-cpu-baseline > /dev/null 2>&1
ls -la $O
