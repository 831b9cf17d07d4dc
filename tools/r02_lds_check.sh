#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp32.py tests/test_gpu_loopback.py -m "gpu and not slow" -x -q > gpurun_out/r02_pytest_lds.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02_pytest_lds.log
python tools/kt.py prof; python tools/kt.py prof fp32
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_sigma$" -c 1 -o gpurun_out/r02_k_sigma_lds python tools/kt.py prof > gpurun_out/r02_ncu_k_sigma.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_pi_contract$" -c 1 -o gpurun_out/r02_k_pi_lds python tools/kt.py prof > gpurun_out/r02_ncu_k_pi.log 2>&1
echo ncu done
