#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_rgf.py tests/test_gpu_guard.py -x -q > gpurun_out/r02_pytest_rgf4.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/r02_pytest_rgf4.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "execute_host or two_streams" > gpurun_out/r02_pytest_e2e.log 2>&1
echo "pytest e2e rc=$?"; tail -1 gpurun_out/r02_pytest_e2e.log
python tools/rgf_time.py rgf_finfet 3
