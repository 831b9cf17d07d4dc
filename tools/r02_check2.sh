#!/bin/bash
# Energy-pair parity cases + the whole -m gpu suite on one GPU, then the default bench line (Π items ordered
# longest-first inside each chunk; separate QT_K_SIGMA_PAIR timing kind).
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r02q_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02q_pytest_gpu.log; grep -E "FAIL|Error" gpurun_out/r02q_pytest_gpu.log | head
timeout 1200 python bench.py > gpurun_out/r02q_bench_cfg3.json 2> gpurun_out/r02q_bench_cfg3.err
echo "bench rc=$?"; head -c 400 gpurun_out/r02q_bench_cfg3.json; echo
