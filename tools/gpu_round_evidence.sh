#!/bin/bash
# Bench + launch list + one full ncu capture of the dominant kernel (k_sigma) at the bench workload.
set -x
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
python tools/time_cfg.py cfg3 1 > gpurun_out/time_cfg3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^k_sigma$" -c 1 -o gpurun_out/prof_sigma_cfg3 \
    python tools/time_cfg.py cfg3 1 > gpurun_out/ncu_sigma_cfg3.log 2>&1
