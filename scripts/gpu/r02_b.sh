set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
for L in 1 all; do STN_DEBUG=lanes=$L timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_v2_$L.json > gpurun_out/steps_cfg5_v2_$L.txt 2>&1; head -3 gpurun_out/steps_cfg5_v2_$L.txt; done
STN_DEBUG=lanes=1,lanes_pf=0 timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_v2_nopf.json > gpurun_out/steps_cfg5_v2_nopf.txt 2>&1; head -3 gpurun_out/steps_cfg5_v2_nopf.txt
STN_DEBUG=lanes=1,lanes_pf=1 timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_v2_pf.json > gpurun_out/steps_cfg5_v2_pf.txt 2>&1; head -3 gpurun_out/steps_cfg5_v2_pf.txt
for L in 0 1 all; do STN_DEBUG=lanes=$L timeout 600 python scripts/step_profile.py cfg2 fast 64 gpurun_out/steps_cfg2_v2_$L.json > gpurun_out/steps_cfg2_v2_$L.txt 2>&1; head -3 gpurun_out/steps_cfg2_v2_$L.txt; done
for L in 0 1; do STN_DEBUG=lanes=$L timeout 600 python scripts/step_profile.py cfg4 fast 4 gpurun_out/steps_cfg4_v2_$L.json > gpurun_out/steps_cfg4_v2_$L.txt 2>&1; head -3 gpurun_out/steps_cfg4_v2_$L.txt; done
timeout 900 python bench.py --config cfg5 > gpurun_out/bench_cfg5_b.json 2> gpurun_out/bench_cfg5_b.err; tail -3 gpurun_out/bench_cfg5_b.err; cat gpurun_out/bench_cfg5_b.json
timeout 600 python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_plain.log 2>&1 && timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_cfg5.csv python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_cfg5.log 2>&1; tail -3 gpurun_out/ncu_cfg5.log
