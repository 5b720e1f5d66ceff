set -x
/usr/bin/time -f "%e s gpu tests" timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 900 python bench.py --config cfg5 > gpurun_out/bench_cfg5_p.json 2> gpurun_out/bench_cfg5_p.err; tail -2 gpurun_out/bench_cfg5_p.err; python -c "import json;j=json.load(open('gpurun_out/bench_cfg5_p.json'));print(j['value'], j['e2e'])"
timeout 1200 python scripts/fast_errors.py gpurun_out/fast_errors.json 2>&1 | tail -12
timeout 900 python bench.py --config cfg4 --cpu-budget 20 > gpurun_out/bench_cfg4_p.json 2> gpurun_out/bench_cfg4_p.err; tail -2 gpurun_out/bench_cfg4_p.err; cut -c1-200 gpurun_out/bench_cfg4_p.json
timeout 900 python bench.py --config cfg2 --cpu-budget 20 > gpurun_out/bench_cfg2_p.json 2> gpurun_out/bench_cfg2_p.err; tail -2 gpurun_out/bench_cfg2_p.err; cut -c1-200 gpurun_out/bench_cfg2_p.json
