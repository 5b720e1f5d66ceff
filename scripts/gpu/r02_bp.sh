set -x
timeout 600 python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_plain_bp.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tcf -c 1 -o gpurun_out/tcf_bp python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_bp.log 2>&1; tail -2 gpurun_out/ncu_bp.log
