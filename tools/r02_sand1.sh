#!/bin/bash
# Σ sandwich: one bulk copy per (pair, energy) slot (scratch rows padded like the ring) instead of nine.
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp32.py -m "gpu and not slow" -q -x > gpurun_out/r02s_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02s_pytest.log; grep FAILED gpurun_out/r02s_pytest.log | head
python tools/kt.py prof; python tools/kt.py prof fp32; python tools/kt.py cfg3
