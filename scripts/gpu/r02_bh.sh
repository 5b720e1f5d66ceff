set -x
timeout 600 python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_plain_bh.log 2>&1 && timeout 2400 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:stn_chain --launch-skip 42 -c 1 -o gpurun_out/chain_bh python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_bh.log 2>&1; tail -3 gpurun_out/ncu_bh.log; ls -la gpurun_out/chain_bh*
