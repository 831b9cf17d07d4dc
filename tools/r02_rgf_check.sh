#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_rgf.py -q -x > gpurun_out/r02_pytest_rgf.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_rgf.log
timeout 600 python tools/rgf_time.py rgf_finfet 3
bash tools/r02_rgf_prof.sh
