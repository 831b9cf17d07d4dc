#!/bin/bash
timeout 2400 python bench.py --gpus 4 --config cfg5 --shard atom --steps 2 --warmup 1 --no-e2e --workspace-gb 4 --fill-halo > gpurun_out/r02f_bench_cfg5_4gpu.json 2> gpurun_out/r02f_bench_cfg5_4gpu.err
echo "cfg5 x4 rc=$?"; head -c 250 gpurun_out/r02f_bench_cfg5_4gpu.json; echo
