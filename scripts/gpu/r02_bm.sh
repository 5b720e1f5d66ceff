set -x
STN_DEBUG=sweep_debug,chain_exp_single=1 timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_bm.json > gpurun_out/steps_cfg5_bm.txt 2>&1; grep -E "slices|rror" gpurun_out/steps_cfg5_bm.txt; python - <<PY
import json
a=json.load(open('gpurun_out/steps_cfg5_bm.json')); n=a['slices']
print([(r['step'], r['kernel'], round(r['ms']/n,3)) for r in a['rows'] if r['step'] in (1155, 649, 1185, 241, 1605, 693, 1083)])
PY
timeout 1500 python scripts/ab_compare.py cfg5 8 3 "" "chain_exp_single=1" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 2 "" "chain_exp_single=1" 2>&1 | grep -E "median|rror"
