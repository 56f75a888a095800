#!/bin/bash
# L1 / L2 throughput breakdown of one launch of the given kernel regex (c4, 40 its)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
K=${K:-k_step}
timeout 600 ncu --clock-control none -k regex:$K -s 5 -c 1 \
  --metrics breakdown:l1tex__throughput.avg.pct_of_peak_sustained_active,breakdown:lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__m_xbar2l1tex_read_bytes.sum,l1tex__m_l1tex2xbar_write_bytes.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__cycles_elapsed.avg,smsp__inst_executed_op_global_ld.sum,l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum,gpu__time_duration.sum \
  --csv python tools/solve_once.py --config c4 --max-m 40 > gpurun_out/ncu_l1_$K.csv 2> gpurun_out/ncu_l1_$K.err
echo EXIT $? >> gpurun_out/ncu_l1_$K.err
