rm -rf gpurun_out; mkdir -p gpurun_out
timeout 600 ncu --kernel-name-base demangled --set full --import-source on --clock-control none -k 'regex:k_absorb_tma<\(int\)8, \(int\)4, \(int\)16' -s 1 -c 1 -o gpurun_out/r37_gather python scripts/ncu_target.py cfg2 1 > gpurun_out/r37_ncu.log 2>&1; echo ncu=$?
STN_TMA_DBG=7 timeout 600 ncu --kernel-name-base demangled --set full --clock-control none -k 'regex:k_absorb_tma<\(int\)8, \(int\)4, \(int\)16' -s 1 -c 1 -o gpurun_out/r37_gather_dbg7 python scripts/ncu_target.py cfg2 1 > gpurun_out/r37_ncu2.log 2>&1; echo ncu=$?
ls -la gpurun_out
