rm -rf gpurun_out; mkdir -p gpurun_out
STN_SWEEP_ONLY=${ONLY:-8} STN_SWEEP_DBG=${DBG:-2} timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 2 -c 1 -o gpurun_out/r21_sweep python scripts/step_profile.py cfg2 > gpurun_out/r21_ncu.log 2>&1; echo ncu=$?
ls -la gpurun_out
