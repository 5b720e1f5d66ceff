set -x
free -g | head -2
date; timeout 1500 python bench.py --impl reference --config cfg5 > gpurun_out/ref_cfg5.json 2> gpurun_out/ref_cfg5.err; date; tail -2 gpurun_out/ref_cfg5.err; cat gpurun_out/ref_cfg5.json
timeout 600 python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_plain_r.log 2>&1 && timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_cfg5_r02.csv python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_r.log 2>&1; tail -1 gpurun_out/ncu_r.log
timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:stn_chain -c 1 -o gpurun_out/chainjit_r python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_r2.log 2>&1; tail -1 gpurun_out/ncu_r2.log
