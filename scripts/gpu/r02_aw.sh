set -x
timeout 900 python bench.py > gpurun_out/bench_cfg5_aw.json 2> gpurun_out/bench_cfg5_aw.err; python -c "
import json; j=json.load(open('gpurun_out/bench_cfg5_aw.json')); print(j['value'], j['ms_per_step'], j['e2e']['value'], j['roofline']['kernel'], j['roofline']['frac'], j['clocks'], j['gpu_launches'])"
timeout 600 python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_plain_aw.log 2>&1 && timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_cfg5_aw.csv python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_aw.log 2>&1; tail -2 gpurun_out/ncu_aw.log
