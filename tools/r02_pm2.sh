#!/bin/bash
# Fixed multi-energy-pair tiles: parity; Π EC=2 variant; FP32 Σ-sandwich ring variants; cfg3 timing.
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "pair or norb_sweep or small_config_sampled or micro or multichunk or deterministic or wide_window or window_sweep or shift_step" > gpurun_out/r02n_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02n_pytest.log; grep FAILED gpurun_out/r02n_pytest.log | head
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cfg3_sampled_integer" > gpurun_out/r02n_pytest_cfg3.log 2>&1
echo "pytest cfg3 rc=$?"; tail -2 gpurun_out/r02n_pytest_cfg3.log
cp paper_1912_10024_b200/libqtsse.so /tmp/libqtsse.cur.so
echo "== cur"; python tools/kt.py prof; python tools/kt.py prof fp32; python tools/kt.py cfg3
for v in piec2s2; do cp variants/$v.so paper_1912_10024_b200/libqtsse.so; echo "== $v"; python tools/kt.py prof; done
for v in sf12x27 sf16x27 sf8x24 sf12x20; do cp variants/$v.so paper_1912_10024_b200/libqtsse.so; echo "== $v"; python tools/kt.py prof fp32; done
cp /tmp/libqtsse.cur.so paper_1912_10024_b200/libqtsse.so
