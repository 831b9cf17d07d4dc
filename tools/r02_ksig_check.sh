#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -m "gpu and not slow" -x -q > gpurun_out/r02_pytest_ks.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02_pytest_ks.log
python tools/kt.py prof; python tools/kt.py prof
python tools/time_cfg.py cfg3 1
