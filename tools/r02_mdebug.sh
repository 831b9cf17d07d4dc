#!/bin/bash
# Bisect the multi-GPU failures of the last 4-GPU run on 2 GPUs: per-rank per-output mismatch counts.
run() { timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=$1 tools/mgpu_debug.py ${@:2} 2>&1 | grep -E "rank|mgpu ok|Error|error" | head -20; }
cp paper_1912_10024_b200/libqtsse.so /tmp/cur.so
echo "== cur prof integer fp32 atom separate"; run 29501 prof integer fp32 atom 0 separate
cp variants/v_b0a6a74.so paper_1912_10024_b200/libqtsse.so
echo "== b0a6a74 (before one-copy) prof integer fp32 atom separate"; run 29502 prof integer fp32 atom 0 separate
cp variants/v_a347b4c.so paper_1912_10024_b200/libqtsse.so
echo "== a347b4c (LPT, before multi tiles) prof integer fp32 atom separate"; run 29503 prof integer fp32 atom 0 separate
cp /tmp/cur.so paper_1912_10024_b200/libqtsse.so
echo "== cur prof random fp64 energy fused"; run 29504 prof random fp64 energy 0 fused
