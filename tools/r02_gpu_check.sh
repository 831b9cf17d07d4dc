#!/bin/bash
# quick GPU check: fast -m gpu tests, then a short bench (no CPU leg)
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/r02_pytest_fast.log 2>&1
echo "pytest rc=$?"
tail -5 gpurun_out/r02_pytest_fast.log
timeout 600 python bench.py --steps 3 --warmup 1 --no-cpu > gpurun_out/r02_bench_quick.json 2> gpurun_out/r02_bench_quick.err
echo "bench rc=$?"
cat gpurun_out/r02_bench_quick.json | head -c 3000
