#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp32.py tests/test_gpu_loopback.py -m "gpu and not slow" -x -q > gpurun_out/r02_pytest_sand.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_sand.log
python tools/kt.py prof; python tools/kt.py prof fp32
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sigma_sand" -c 1 -o gpurun_out/r02_sand_v2 python tools/kt.py prof > gpurun_out/r02_ncu_sand_v2.log 2>&1
echo ncu rc=$?
