#!/bin/bash
# ncu --set full of the two sandwich kernels (k_sigma_sand, k_pi_w) on the profiling slice (cfg3 per-atom shape).
set -x
python tools/time_cfg.py prof 2 > gpurun_out/r02_time_prof.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sigma_sand" -c 1 -o gpurun_out/r02_sand \
    python tools/time_cfg.py prof 1 > gpurun_out/r02_ncu_sand.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pi_w" -c 1 -o gpurun_out/r02_piw \
    python tools/time_cfg.py prof 1 > gpurun_out/r02_ncu_piw.log 2>&1
ls -la gpurun_out
