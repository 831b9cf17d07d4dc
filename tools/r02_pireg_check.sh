#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -m "gpu and not slow" -x -q > gpurun_out/r02_pytest_pireg.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/r02_pytest_pireg.log
python tools/kt.py prof; python tools/kt.py prof
bash tools/run_variants.sh prof pi_oldcontract
