#!/bin/bash
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:"k_sigma_pair" -c 12 --log-file gpurun_out/r02w_pair_traffic_cfg3.csv python tools/time_cfg.py cfg3 1 > gpurun_out/r02w_ncu_traffic.log 2>&1
echo "ncu rc=$?"
