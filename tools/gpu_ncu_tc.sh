#!/bin/bash
# per-launch metrics of every tensor-core conv launch of one r18 step (small report)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,launch__grid_size,sm__cycles_active.avg,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__inst_executed_pipe_tma.sum
timeout 900 ncu --metrics $M --clock-control none --cache-control none --kernel-name-base demangled \
  -k "regex:conv_tc_kernel|conv_pair|splitk_finish" -c 120 --csv --log-file gpurun_out/${1:-r2_tc34}.csv python tools/profile_step.py 1 > /dev/null 2>&1
echo rc=$?
