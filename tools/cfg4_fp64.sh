#!/bin/bash
# cfg4 (BASELINE config 4) on N GPUs in FP64: atom sharding (default) and energy sharding, 3 + 3 steps each.
N=${1:-4}; P=29611
for sh in atom energy; do
  P=$((P+1))
  torchrun --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --config cfg4 \
    --shard $sh --no-e2e --no-cpu --workspace-gb 24 > gpurun_out/bench_cfg4_fp64_${sh}_${N}gpu.json 2> gpurun_out/bench_cfg4_fp64_${sh}_${N}gpu.err
  tail -1 gpurun_out/bench_cfg4_fp64_${sh}_${N}gpu.err | cut -c1-200
  cut -c1-200 gpurun_out/bench_cfg4_fp64_${sh}_${N}gpu.json
done
