rm -rf gpurun_out; mkdir -p gpurun_out
STN_PLAN_DUMP=1 timeout 300 python scripts/ncu_target.py cfg2 1 > gpurun_out/r65_dump.txt 2>&1; echo dump=$?
timeout 900 python bench.py > gpurun_out/r65_bench.json 2> gpurun_out/r65_bench.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r65_launches.csv python scripts/ncu_target.py cfg2 1 > gpurun_out/r65_l.log 2>&1; echo ncu=$?
timeout 900 ncu --kernel-name-base demangled --set full --import-source on --clock-control none -k 'regex:k_absorb_direct<\(bool\)0, \(int\)16, \(int\)8, \(bool\)1>' -s 2 -c 1 -o gpurun_out/r65_direct python scripts/ncu_target.py cfg2 1 > gpurun_out/r65_ncu1.log 2>&1; echo ncu1=$?
ls -la gpurun_out
