rm -rf gpurun_out; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:${KRE:-absorb_mmaILi4} -s 2 -c 1 -o gpurun_out/r24_mma python scripts/step_profile.py cfg2 > gpurun_out/r24_ncu.log 2>&1; echo ncu=$?
ls -la gpurun_out
