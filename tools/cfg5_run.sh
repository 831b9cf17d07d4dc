#!/bin/bash
# cfg5 (BASELINE config 5: 10,240 atoms, NE=1000, Nω=70, Nkz=Nqz=5; 24.7 Pflop per step) on N GPUs,
# atom sharding: FP32 mixed mode and FP64, 3 + 3 steps each.
N=${1:-4}; P=29711
for pr in fp32 fp64; do
  P=$((P+1))
  torchrun --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --config cfg5 \
    --precision $pr --no-e2e --no-cpu --workspace-gb 16 > gpurun_out/bench_cfg5_${pr}_${N}gpu.json 2> gpurun_out/bench_cfg5_${pr}_${N}gpu.err
  grep -iE "error|memory" gpurun_out/bench_cfg5_${pr}_${N}gpu.err | head -3
  cut -c1-200 gpurun_out/bench_cfg5_${pr}_${N}gpu.json
done
