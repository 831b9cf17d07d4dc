#!/bin/bash
# 2-GPU check: multi-GPU parity (real NCCL), then bench --gpus 2 self-launch (atom, energy)
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/r02_pytest_2gpu.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/r02_pytest_2gpu.log
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/r02_bench_2gpu_atom.json 2> gpurun_out/r02_bench_2gpu_atom.err
echo "bench atom rc=$?"; head -c 1500 gpurun_out/r02_bench_2gpu_atom.json
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 1 --no-cpu --no-e2e --shard energy > gpurun_out/r02_bench_2gpu_energy.json 2> gpurun_out/r02_bench_2gpu_energy.err
echo "bench energy rc=$?"; head -c 1500 gpurun_out/r02_bench_2gpu_energy.json
