#!/bin/bash
# 4-GPU evidence: multi-GPU parity (2 x 2 grid included), cfg3 bench at N=4 (atom), cfg4 energy-sharded and 2-D
timeout 1500 python -m pytest tests/test_multigpu.py -q -rs > gpurun_out/r02_pytest_4gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_4gpu.log
timeout 900 python bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r02_bench_cfg3_4gpu.json 2> gpurun_out/r02_bench_cfg3_4gpu.err
echo "bench cfg3 x4 rc=$?"; head -c 300 gpurun_out/r02_bench_cfg3_4gpu.json; echo
timeout 1500 python bench.py --gpus 4 --config cfg4 --shard energy --steps 2 --warmup 1 --no-e2e --workspace-gb 16 > gpurun_out/r02_bench_cfg4_4gpu_energy.json 2> gpurun_out/r02_bench_cfg4_4gpu_energy.err
echo "bench cfg4 energy x4 rc=$?"; head -c 300 gpurun_out/r02_bench_cfg4_4gpu_energy.json; echo
timeout 1500 python bench.py --gpus 4 --config cfg4 --shard 2d --grid-atoms 2 --steps 2 --warmup 1 --no-e2e --workspace-gb 16 > gpurun_out/r02_bench_cfg4_4gpu_2d.json 2> gpurun_out/r02_bench_cfg4_4gpu_2d.err
echo "bench cfg4 2d x4 rc=$?"; head -c 300 gpurun_out/r02_bench_cfg4_4gpu_2d.json; echo
