rm -rf gpurun_out; mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"absorb_mma|absorb_tc|k_gemm_tc|k_split_a|k_absorb3|k_absorb2" -c 16 -o gpurun_out/r30_full python scripts/ncu_target.py cfg2 1 > gpurun_out/r30_ncu.log 2>&1; echo ncu=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r30_launches.csv python scripts/ncu_target.py cfg2 1 > gpurun_out/r30_l.log 2>&1; echo ncu2=$?
tail -3 gpurun_out/r30_ncu.log
ls -la gpurun_out
