set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg5 or fast" 2>&1 | tail -2
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_bc.json > gpurun_out/steps_cfg5_bc.txt 2>&1; grep -E "slices|rror" gpurun_out/steps_cfg5_bc.txt; python - <<PY
import json
j=json.load(open('gpurun_out/steps_cfg5_bc.json')); n=j['slices']
print([(r['step'], r['kernel'], round(r['ms']/n,3)) for r in j['rows'] if r['step'] in (259, 816, 1306, 1394)])
PY
timeout 1200 python scripts/ab_compare.py cfg5 8 3 "tcf_gather=0" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 2 "tcf_gather=0" "" 2>&1 | grep -E "median|rror"
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
