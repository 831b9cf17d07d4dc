#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py tests/test_gpu_guard.py -m "gpu and not slow" -x -q > gpurun_out/r02_pytest_split.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/r02_pytest_split.log
python tools/kt.py prof; python tools/kt.py prof
timeout 900 python tools/time_cfg.py cfg3_norb12 1 > gpurun_out/r02_time_cfg3_norb12.log 2>&1; tail -1 gpurun_out/r02_time_cfg3_norb12.log
