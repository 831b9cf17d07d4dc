#!/bin/bash
# cfg4 (BASELINE config 4: 4,864 atoms, NE=706, Nω=70, Nkz=Nqz=7) atom-sharded on N GPUs, FP64 and FP32 modes.
N=${1:-4}
torchrun --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus $N --config cfg4 \
  --steps 3 --warmup 3 --precision fp32 --no-e2e --workspace-gb 24 > gpurun_out/bench_cfg4_fp32_${N}gpu.json 2> gpurun_out/bench_cfg4_fp32_${N}gpu.err
tail -2 gpurun_out/bench_cfg4_fp32_${N}gpu.err
torchrun --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus $N --config cfg4 \
  --steps 1 --warmup 1 --no-e2e --workspace-gb 24 > gpurun_out/bench_cfg4_fp64_${N}gpu.json 2> gpurun_out/bench_cfg4_fp64_${N}gpu.err
tail -2 gpurun_out/bench_cfg4_fp64_${N}gpu.err
cut -c1-300 gpurun_out/bench_cfg4_*_${N}gpu.json
