#!/bin/bash
# DRAM bytes of every k_sigma launch of one qt_sse_sigma call at cfg3 (2 metrics only), then a full-set
# capture of one k_sigma launch on the profiling slice.
python tools/kt.py cfg3 > gpurun_out/kt_cfg3.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"^k_sigma$" \
    --csv --log-file gpurun_out/traffic_cfg3.csv python tools/kt.py cfg3 > gpurun_out/ncu_traffic.log 2>&1
python tools/kt.py prof > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^k_sigma$" -c 1 -o gpurun_out/prof_sigma_v6 \
    python tools/kt.py prof > gpurun_out/ncu_s6.log 2>&1
