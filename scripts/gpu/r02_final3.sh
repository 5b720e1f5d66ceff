set -x
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_cfg5_f3.json 2> gpurun_out/bench_cfg5_f3.err; python -c "
import json; j=json.load(open('gpurun_out/bench_cfg5_f3.json')); r=j['roofline']; print('cfg5', j['value'], j['ms_per_step'], j['e2e']['value'], r['kernel'], round(r['frac'],3), r['traffic'], (j.get('cpu_baseline') or {}).get('value'), j['clocks'], j['gpu_launches'])"
