#!/bin/bash
# final multi-GPU evidence: cfg3 at 2 and 4 GPUs (atom grid), cfg5 (10,240 atoms, NE = 1000, Nkz = 5) atom-sharded on 4
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r02f_bench_cfg3_2gpu.json 2> gpurun_out/r02f_bench_cfg3_2gpu.err
echo "cfg3 x2 rc=$?"; head -c 250 gpurun_out/r02f_bench_cfg3_2gpu.json; echo
timeout 900 python bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r02f_bench_cfg3_4gpu.json 2> gpurun_out/r02f_bench_cfg3_4gpu.err
echo "cfg3 x4 rc=$?"; head -c 250 gpurun_out/r02f_bench_cfg3_4gpu.json; echo
timeout 2400 python bench.py --gpus 4 --config cfg5 --shard atom --steps 2 --warmup 1 --no-e2e --workspace-gb 4 --fill-halo > gpurun_out/r02f_bench_cfg5_4gpu.json 2> gpurun_out/r02f_bench_cfg5_4gpu.err
echo "cfg5 x4 rc=$?"; head -c 250 gpurun_out/r02f_bench_cfg5_4gpu.json; echo
