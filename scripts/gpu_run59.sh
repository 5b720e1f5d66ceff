rm -rf gpurun_out; mkdir -p gpurun_out
timeout 300 python scripts/step_profile.py cfg2 > gpurun_out/r59_prof.txt 2>&1; echo prof=$?
timeout 1200 python bench.py > gpurun_out/r59_bench.log 2>&1; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r59_launches.csv python scripts/ncu_target.py cfg2 1 > gpurun_out/r59_l.log 2>&1; echo ncu=$?
timeout 900 ncu --kernel-name-base demangled --set full --import-source on --clock-control none -k 'regex:k_absorb_direct<\(bool\)0, \(int\)16, \(int\)16, \(bool\)1>' -s 2 -c 1 -o gpurun_out/r59_direct python scripts/ncu_target.py cfg2 1 > gpurun_out/r59_ncu1.log 2>&1; echo ncu1=$?
timeout 900 ncu --kernel-name-base demangled --set full --import-source on --clock-control none -k 'regex:k_absorb_tma<\(int\)32, \(int\)1, \(int\)128' -c 1 -o gpurun_out/r59_tma python scripts/ncu_target.py cfg2 1 > gpurun_out/r59_ncu2.log 2>&1; echo ncu2=$?
timeout 900 ncu --kernel-name-base demangled --set full --import-source on --clock-control none -k 'regex:k_gemm_tc256' -s 1 -c 1 -o gpurun_out/r59_gemm python scripts/ncu_target.py cfg2 1 > gpurun_out/r59_ncu3.log 2>&1; echo ncu3=$?
ls -la gpurun_out; grep "^{" gpurun_out/r59_bench.log | cut -c1-200
