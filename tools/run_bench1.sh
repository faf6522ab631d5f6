set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python bench.py > gpurun_out/bench_r1a.json 2> gpurun_out/bench_r1a.err; tail -3 gpurun_out/bench_r1a.err
cat gpurun_out/bench_r1a.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1a.csv python bench.py --steps 2 --warmup 3 --no-verify --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_modexp -s 3 -c 1 -o gpurun_out/prof_r1a python bench.py --steps 1 --warmup 3 --no-verify --no-cpu-baseline > gpurun_out/ncu_r1a.log 2>&1
tail -5 gpurun_out/ncu_r1a.log
ls -la gpurun_out
