#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_rgf.py -x -q > gpurun_out/r02_pytest_rgf3.log 2>&1
echo "pytest rgf rc=$?"; tail -1 gpurun_out/r02_pytest_rgf3.log
python tools/rgf_time.py rgf_finfet 2
python tools/kt.py prof
bash tools/run_variants.sh prof sandsplit sandsplit_w8
