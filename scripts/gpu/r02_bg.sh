set -x
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_bg.json > gpurun_out/steps_cfg5_bg.txt 2>&1; grep -E "slices|rror|steps 1365" gpurun_out/steps_cfg5_bg.txt | head
python - <<PY
import json
j=json.load(open('gpurun_out/steps_cfg5_bg.json')); n=j['slices']
print([(r['step'], r['kernel'], round(r['ms']/n,3)) for r in j['rows'] if r['step'] in (1365, 1306, 1394, 259, 816)])
PY
timeout 1500 python scripts/ab_compare.py cfg5 8 3 "" "tcf=2" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 3 "" "tcf=2" 2>&1 | grep -E "median|rror"
