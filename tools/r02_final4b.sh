#!/bin/bash
# Final round-2 evidence (last build) on a 4-GPU box: full -m gpu suite (1-, 2- and 4-GPU cases), smoke, the
# default bench line on one GPU, bench --gpus 2 / 4, the ncu launch list, one full ncu capture of k_sigma_pair at
# cfg3 and the DRAM bytes of 20 of its launches (the bench roofline traffic).
timeout 3000 python -m pytest tests -m gpu -q -rs > gpurun_out/r02x_pytest_gpu_4gpubox.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02x_pytest_gpu_4gpubox.log; grep FAILED gpurun_out/r02x_pytest_gpu_4gpubox.log | head
CUDA_VISIBLE_DEVICES=0 timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02x_smoke.log 2>&1; echo "smoke rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 1200 python bench.py > gpurun_out/r02x_bench_cfg3.json 2> gpurun_out/r02x_bench_cfg3.err
echo "bench x1 rc=$?"; head -c 200 gpurun_out/r02x_bench_cfg3.json; echo
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r02x_bench_cfg3_2gpu.json 2> gpurun_out/r02x_bench_cfg3_2gpu.err
echo "bench x2 rc=$?"; head -c 200 gpurun_out/r02x_bench_cfg3_2gpu.json; echo
timeout 900 python bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r02x_bench_cfg3_4gpu.json 2> gpurun_out/r02x_bench_cfg3_4gpu.err
echo "bench x4 rc=$?"; head -c 200 gpurun_out/r02x_bench_cfg3_4gpu.json; echo
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02x_launches_cfg3.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02x_ncu_launch.log 2>&1
echo "ncu launch rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sigma_pair" -c 1 -o gpurun_out/r02x_k_sigma_pair_cfg3 \
    python tools/time_cfg.py cfg3 1 > gpurun_out/r02x_ncu_pair.log 2>&1
echo "ncu pair rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:"k_sigma_pair" -c 20 --log-file gpurun_out/r02x_pair_traffic_cfg3.csv python tools/time_cfg.py cfg3 1 > gpurun_out/r02x_ncu_traffic.log 2>&1
echo "ncu traffic rc=$?"
