set -x
timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_bq.json > gpurun_out/steps_cfg5_bq.txt 2>&1; grep -E "slices|rror" gpurun_out/steps_cfg5_bq.txt; python - <<PY
import json
j=json.load(open('gpurun_out/steps_cfg5_bq.json')); n=j['slices']
print([(r['step'], r['kernel'], round(r['ms']/n,3)) for r in j['rows'] if r['kernel']=='gemm_tc'])
PY
timeout 600 python scripts/step_profile.py cfg4 fast 4 gpurun_out/steps_cfg4_bq.json > /dev/null 2>&1; python - <<PY
import json
j=json.load(open('gpurun_out/steps_cfg4_bq.json')); n=j['slices']
print([(r['step'], r['kernel'], round(r['ms']/n,3)) for r in j['rows'] if r['kernel']=='gemm_tc'])
PY
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg5 or 53" 2>&1 | tail -2
