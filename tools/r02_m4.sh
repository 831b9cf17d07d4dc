#!/bin/bash
# Re-run on 4 GPUs the multi-GPU cases that failed / hung in r02x (each under its own SIGTERM timeout so torchrun
# stops its workers), then bench --gpus 4.
run() { n=$1; port=$2; shift 2
  timeout -s TERM 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$port tests/mgpu_worker.py "$@" > gpurun_out/r02w_mgpu_$port.log 2>&1
  echo "rc=$? n=$n $*"; grep -E "mgpu ok|Error|assert" gpurun_out/r02w_mgpu_$port.log | head -5; }
run 2 29611 prof integer fp32 atom 0 separate
run 2 29612 prof random fp32 energy 0 fused
run 4 29613 small integer fp64 2d 2 fused
run 4 29614 prof random fp64 2d 2 fused
run 4 29615 small integer fp32 2d 2 fused
nvidia-smi --query-compute-apps=pid,used_memory --format=csv
timeout 600 python bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu > gpurun_out/r02w_bench_cfg3_4gpu.json 2> gpurun_out/r02w_bench_cfg3_4gpu.err
echo "bench x4 rc=$?"; head -c 200 gpurun_out/r02w_bench_cfg3_4gpu.json; echo
