set -x
timeout 600 python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_plain_ba.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tcf -c 3 -o gpurun_out/tcf_ba python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_ba.log 2>&1; tail -3 gpurun_out/ncu_ba.log; ls -la gpurun_out/tcf_ba*
