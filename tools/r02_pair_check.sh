#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py tests/test_gpu_guard.py -m "gpu and not slow" -x -q > gpurun_out/r02_pytest_pair.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/r02_pytest_pair.log
python tools/kt.py prof; python tools/kt.py prof
bash tools/run_variants.sh prof nopair
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg3_sampled_integer or small_config_sampled" > gpurun_out/r02_pytest_pair_cfg3.log 2>&1
echo "cfg3 integer rc=$?"; tail -1 gpurun_out/r02_pytest_pair_cfg3.log
