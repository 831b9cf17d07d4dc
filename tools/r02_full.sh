#!/bin/bash
# Round-2 evidence on one B200: full -m gpu suite, the default bench line, the ncu launch list of the same
# command, and one ncu --set full capture of the dominant kernel at the bench workload (DRAM traffic).
timeout 3000 python -m pytest tests -m gpu -q -rs > gpurun_out/r02_pytest_gpu_full.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_gpu_full.log
timeout 1200 python bench.py > gpurun_out/r02_bench_cfg3.json 2> gpurun_out/r02_bench_cfg3.err
echo "bench rc=$?"; head -c 400 gpurun_out/r02_bench_cfg3.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg3.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02_ncu_launch.log 2>&1
echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_sigma$" -c 1 -o gpurun_out/r02_k_sigma_cfg3 \
    python tools/time_cfg.py cfg3 1 > gpurun_out/r02_ncu_sigma_cfg3.log 2>&1
echo "ncu full rc=$?"
