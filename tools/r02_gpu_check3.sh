#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -s -k "shift_step or deterministic or long_contraction or multichunk or fused or loopback or fp32" > gpurun_out/r02_pytest_new.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|Error|FP32 mode|assert" gpurun_out/r02_pytest_new.log | tail -20
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --precision fp32 > gpurun_out/r02_bench_fp32_quick.json 2> gpurun_out/r02_bench_fp32_quick.err
echo "bench rc=$?"; head -c 600 gpurun_out/r02_bench_fp32_quick.json; grep -o '"kernels_ms_per_step[^}]*}' gpurun_out/r02_bench_fp32_quick.json
