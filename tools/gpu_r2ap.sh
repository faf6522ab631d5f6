#!/bin/bash
# round-2 GPU batch AP: launch list of the C5 bench (Miller-Rabin: setup / rounds / final shares)
O=gpurun_out/r2ap; mkdir -p $O
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv python bench.py --workload c5 --steps 2 --warmup 3 --no-verify --no-identity --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py $O/launches_c5.csv
