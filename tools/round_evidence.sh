#!/bin/bash
# One GPU call: bench (cfg3), the ncu launch list of a 1+1-step bench, k_sigma DRAM traffic at cfg3
# (2 metrics over all launches of one qt_sse_sigma call), and a full-set capture of k_sigma on the
# profiling slice (same per-atom shape; the full set on a cfg3 launch takes ~45 min).
tag=${1:-cur}
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_$tag.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"^k_sigma$" --csv --log-file gpurun_out/traffic_$tag.csv python tools/kt.py cfg3 > gpurun_out/ncu_traffic_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"^k_sigma$" -c 1 -o gpurun_out/prof_sigma_$tag \
    python tools/kt.py prof > gpurun_out/ncu_full_$tag.log 2>&1
ncu -i gpurun_out/prof_sigma_$tag.ncu-rep --page source --csv > gpurun_out/src_$tag.csv 2>/dev/null
ncu -i gpurun_out/prof_sigma_$tag.ncu-rep --page raw --csv > gpurun_out/raw_$tag.csv 2>/dev/null
ls -la gpurun_out/ | tail -20
