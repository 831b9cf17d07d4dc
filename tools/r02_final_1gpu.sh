#!/bin/bash
# Final round-2 single-GPU lines (last build): FP32 mixed mode, RGF workload, the reference arm (CPU oracle),
# and ncu captures of the two sandwich kernels on the profiling slice.
timeout 900 python bench.py --precision fp32 --steps 5 --warmup 3 --no-cpu > gpurun_out/r02y_bench_cfg3_fp32.json 2> gpurun_out/r02y_bench_cfg3_fp32.err
echo "bench fp32 rc=$?"; head -c 250 gpurun_out/r02y_bench_cfg3_fp32.json; echo
timeout 900 python bench.py --workload rgf --steps 5 --warmup 3 > gpurun_out/r02y_bench_rgf.json 2> gpurun_out/r02y_bench_rgf.err
echo "bench rgf rc=$?"; head -c 250 gpurun_out/r02y_bench_rgf.json; echo
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02y_bench_reference.json 2> gpurun_out/r02y_bench_reference.err
echo "reference rc=$?"; head -c 250 gpurun_out/r02y_bench_reference.json; echo
for k in k_sigma_sand k_pi_contract; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$k\$" -c 1 -o gpurun_out/r02y_$k python tools/kt.py prof > gpurun_out/r02y_ncu_$k.log 2>&1
  echo "ncu $k rc=$?"
done
