set -x
timeout 1500 python scripts/ab_compare.py cfg5 8 3 "" "chain_exp_pen=0" 2>&1 | grep -E "median|rror"
STN_DEBUG=sweep_debug,chain_exp_pen=0 timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_bs.json > gpurun_out/steps_cfg5_bs.txt 2>&1; grep -E "slices|steps 1155" gpurun_out/steps_cfg5_bs.txt | head -3; python - <<PY
import json
j=json.load(open('gpurun_out/steps_cfg5_bs.json')); n=j['slices']
print([(r['step'], r['kernel'], round(r['ms']/n,3)) for r in j['rows'] if r['step'] in (1155, 1161, 1170)])
PY
