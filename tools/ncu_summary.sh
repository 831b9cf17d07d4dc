#!/bin/bash
# usage: tools/ncu_summary.sh rep.ncu-rep  -> key metrics + stall summary
rep=$1
ncu -i $rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for k in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_bytes.sum','sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_tensor_subpipe_dmma.sum','sm__warps_active.avg.pct_of_peak_sustained_active','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','smsp__inst_executed.sum','sm__cycles_elapsed.avg']:
  for i,x in enumerate(h):
    if x==k: print('  ',k, v[i], r[1][i])
"
ncu -i $rep --page source --csv --print-source sass 2>/dev/null > /tmp/_src.csv
python $(dirname $0)/ncu_stalls.py /tmp/_src.csv ${2:-10}
