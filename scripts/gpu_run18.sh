rm -rf gpurun_out; mkdir -p gpurun_out
STN_SWEEP_DEBUG=1 timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/r18_prof.txt 2>&1; echo prof=$?
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,smsp__inst_executed_op_global_ld.sum
timeout 900 ncu --clock-control none --section WarpStateStats --section Occupancy --metrics $M -k regex:k_sweep -s 76 -c 19 --csv --page details python scripts/step_profile.py cfg2 > gpurun_out/r18_ncu.csv 2> gpurun_out/r18_ncu.err; echo ncu=$?
grep -c k_sweep gpurun_out/r18_ncu.csv
