set -x
for c in cfg5 cfg4 cfg2; do timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_f1.json 2> gpurun_out/bench_${c}_f1.err; python -c "
import json; j=json.load(open('gpurun_out/bench_${c}_f1.json')); r=j['roofline']; print('$c', j['value'], j['ms_per_step'], j['e2e']['value'], r['kernel'], round(r['frac'],3), (j.get('cpu_baseline') or {}).get('value'), j['clocks'])"; done
timeout 900 python scripts/fast_errors.py gpurun_out/fast_errors_f1.json 2>&1 | tail -2
timeout 600 python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_plain_f1.log 2>&1 && timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_cfg5_f1.csv python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_f1.log 2>&1; tail -1 gpurun_out/ncu_f1.log
