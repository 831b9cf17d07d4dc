#!/bin/bash
# Final round-2 evidence on one B200 (driver-equivalent commands): full -m gpu suite, smoke, the default bench line,
# the FP32 and RGF lines, the ncu launch list of the default bench command, ncu --set full of the top kernels.
timeout 3000 python -m pytest tests -m gpu -q -rs > gpurun_out/r02f_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02f_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r02f_smoke.log
timeout 1200 python bench.py > gpurun_out/r02f_bench_cfg3.json 2> gpurun_out/r02f_bench_cfg3.err
echo "bench rc=$?"; head -c 300 gpurun_out/r02f_bench_cfg3.json; echo
timeout 900 python bench.py --precision fp32 --steps 3 --warmup 2 --no-cpu > gpurun_out/r02f_bench_cfg3_fp32.json 2> gpurun_out/r02f_bench_cfg3_fp32.err
echo "bench fp32 rc=$?"
timeout 900 python bench.py --workload rgf --steps 5 --warmup 2 > gpurun_out/r02f_bench_rgf.json 2> gpurun_out/r02f_bench_rgf.err
echo "bench rgf rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02f_bench_reference.json 2> gpurun_out/r02f_bench_reference.err
echo "reference rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launches_cfg3.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02f_ncu_launch.log 2>&1
echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_sigma$" -c 1 -o gpurun_out/r02f_k_sigma_cfg3 \
    python tools/time_cfg.py cfg3 1 > gpurun_out/r02f_ncu_sigma.log 2>&1
echo "ncu k_sigma rc=$?"
for k in k_sigma_sand k_pi_w2 k_pi_contract; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$k\$" -c 1 -o gpurun_out/r02f_$k python tools/kt.py prof > gpurun_out/r02f_ncu_$k.log 2>&1
  echo "ncu $k rc=$?"
done
