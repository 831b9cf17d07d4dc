#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -x -q -s -k "shift_step or deterministic or long_contraction or multichunk or fused or loopback" > gpurun_out/r02_pytest_new.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|error|FP32 mode" gpurun_out/r02_pytest_new.log | tail -8
