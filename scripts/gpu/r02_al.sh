set -x
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_cfg5_al.json 2> gpurun_out/bench_cfg5_al.err; tail -1 gpurun_out/bench_cfg5_al.err
timeout 900 python bench.py --config cfg4 > gpurun_out/bench_cfg4_al.json 2> gpurun_out/bench_cfg4_al.err; tail -1 gpurun_out/bench_cfg4_al.err
for c in cfg5 cfg4; do python -c "
import json; j=json.load(open('gpurun_out/bench_${c}_al.json')); print('$c', j['value'], j['e2e']['value'], j['roofline']['kernel'], round(j['roofline']['frac'],3), (j.get('cpu_baseline') or {}).get('value'), j['clocks'])"; done
timeout 900 python scripts/fast_errors.py gpurun_out/fast_errors_al.json 2>&1 | tail -8
timeout 600 python scripts/ncu_target.py cfg4 1 > gpurun_out/ncu_target_cfg4_plain.log 2>&1; echo plain rc $?
