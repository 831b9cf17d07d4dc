#!/bin/bash
timeout 380 python -m pytest tests/test_multigpu.py -m gpu -v -rfs > gpurun_out/r02w_pytest_multigpu.log 2>&1
echo "rc=$?"; grep -cE "PASSED" gpurun_out/r02w_pytest_multigpu.log; tail -3 gpurun_out/r02w_pytest_multigpu.log
