#!/bin/bash
# Multi-energy-pair tiles for items of 1..3 pairs in k_sigma_pair (QT_PAIR_MIN = 1) vs k_sigma's multi-energy
# tiles (variant pairmin4): parity, then per-kernel times on the profiling slice and at cfg3.
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pair or norb_sweep or small_config_sampled or micro or multichunk or deterministic" > gpurun_out/r02m_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02m_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cfg3_sampled_integer" > gpurun_out/r02m_pytest_cfg3.log 2>&1
echo "pytest cfg3 rc=$?"; tail -2 gpurun_out/r02m_pytest_cfg3.log
cp paper_1912_10024_b200/libqtsse.so /tmp/libqtsse.cur.so
for v in cur pairmin4; do
  [ "$v" != cur ] && cp variants/$v.so paper_1912_10024_b200/libqtsse.so
  echo "== $v"; python tools/kt.py prof; python tools/kt.py cfg3
  cp /tmp/libqtsse.cur.so paper_1912_10024_b200/libqtsse.so
done
# one full capture of the FP32-mode Σ sandwich (profiling slice) for its stall breakdown
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sigma_sand" -c 1 -o gpurun_out/r02m_k_sigma_sand_fp32 \
    python tools/kt.py prof fp32 > gpurun_out/r02m_ncu_sand32.log 2>&1
echo "ncu rc=$?"
