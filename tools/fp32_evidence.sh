#!/bin/bash
# FP32 mixed mode evidence at cfg3: ncu launch list of a 1+1-step bench, k_sigma_tc DRAM traffic per launch.
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fp32.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --precision fp32 > gpurun_out/ncu_launch_fp32.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"^k_sigma_tc$" --csv --log-file gpurun_out/traffic_fp32.csv python tools/kt.py cfg3 fp32 > gpurun_out/ncu_traffic_fp32.log 2>&1
ls -la gpurun_out/*fp32*
