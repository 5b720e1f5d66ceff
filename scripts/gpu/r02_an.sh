set -x
for i in 1 2; do timeout 900 python bench.py > gpurun_out/bench_cfg5_an$i.json 2> gpurun_out/bench_cfg5_an$i.err; python -c "
import json; j=json.load(open('gpurun_out/bench_cfg5_an$i.json')); print(j['value'], j['ms_per_step'], j['e2e']['value'], j['clocks'])"; done
STN_DEBUG=side=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg2 or cfg1 or streams" 2>&1 | tail -2
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg4 fast 4 gpurun_out/steps_cfg4_an.json > gpurun_out/steps_cfg4_an.txt 2>&1; sed -n '/step kernel/,+6p' gpurun_out/steps_cfg4_an.txt
