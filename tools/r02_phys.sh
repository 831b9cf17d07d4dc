#!/bin/bash
# PHYSICAL input envelope on the GPU (generator bit-equality, FP64 / FP32 parity), a bench line on it, and the DRAM
# traffic of the small-item k_sigma launches beside k_sigma_pair at cfg3 (for the roofline traffic figure).
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp32.py -m gpu -q -rs -k "physical or generator" \
    > gpurun_out/r02p_pytest_physical.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02p_pytest_physical.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --inputs physical > gpurun_out/r02p_bench_cfg3_physical.json \
    2> gpurun_out/r02p_bench_cfg3_physical.err
echo "bench rc=$?"; head -c 300 gpurun_out/r02p_bench_cfg3_physical.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:"^k_sigma" -c 60 --log-file gpurun_out/r02p_sigma_traffic_cfg3.csv python tools/time_cfg.py cfg3 1 \
    > gpurun_out/r02p_ncu_traffic.log 2>&1
echo "ncu rc=$?"
