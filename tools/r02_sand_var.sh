#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp32.py -m "gpu and not slow" -x -q > gpurun_out/r02_pytest_sand.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_sand.log
python tools/kt.py prof; python tools/kt.py prof fp32
bash tools/run_variants.sh prof sandw4s6 sandw8s10 sandw12s16 sandw3s5
