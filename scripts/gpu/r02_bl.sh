set -x
timeout 600 python scripts/ncu_target.py cfg4 1 > gpurun_out/ncu_plain_bl.log 2>&1 && timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc256m -c 4 -o gpurun_out/gemm_bl2 python scripts/ncu_target.py cfg4 1 > gpurun_out/ncu_bl.log 2>&1; tail -2 gpurun_out/ncu_bl.log; ls -la gpurun_out/gemm_bl2*
