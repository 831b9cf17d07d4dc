#!/bin/bash
# tensor-pipe / L2 / smem summary of the FP32-mode tcgen05 kernels on the profiling slice
python tools/kt.py prof fp32 > /dev/null 2>&1
for k in k_sigma_tc k_pi_contract_tc; do
  ncu --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -k regex:"^$k\$" -c 1 --csv python tools/kt.py prof fp32 2>/dev/null | grep -E "^\"[0-9]" | awk -F'","' '{print $5, $(NF-2), $NF}'
done
