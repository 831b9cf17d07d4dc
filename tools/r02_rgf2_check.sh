#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_rgf.py tests/test_gpu_fp32.py tests/test_gpu_guard.py -m "gpu and not slow" -x -q > gpurun_out/r02_pytest_rgf2.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02_pytest_rgf2.log
python tools/rgf_time.py rgf_finfet 3
python tools/kt.py prof fp32; bash tools/run_variants.sh prof piw_old; 
cp variants/piw_old.so /tmp/x.so
