set -x
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/bench_final_x.json 2> gpurun_out/bench_final_x.err; tail -2 gpurun_out/bench_final_x.err; python -c "
import json; j=json.load(open('gpurun_out/bench_final_x.json')); print(j['value'], j['e2e']['value'], j['e2e']['one_time_setup_s'], j['roofline']['kernel'], j['roofline']['frac'], j['roofline']['traffic'], j['cpu_baseline']['value'], j['clocks'])"
