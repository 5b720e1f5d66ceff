rm -rf gpurun_out; mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none -k regex:"absorb_mma|absorb_tc|k_gemm_tc" -c 8 -o gpurun_out/r31_full python scripts/ncu_target.py cfg2 1 > gpurun_out/r31_ncu.log 2>&1; echo ncu=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r31_launches.csv python scripts/ncu_target.py cfg2 1 > gpurun_out/r31_l.log 2>&1; echo ncu2=$?
tail -3 gpurun_out/r31_ncu.log
ls -la gpurun_out
