set -x
timeout 1500 python scripts/ab_compare.py cfg5 8 3 "" "chain_wreg_exp=16" "chain_wreg_exp=48" 2>&1 | grep -E "median|rror"
for v in "chain_wreg_exp=16" "chain_wreg_exp=48"; do STN_DEBUG=$v timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_bk_$v.json > /dev/null 2>&1; python - <<PY
import json
j=json.load(open('gpurun_out/steps_cfg5_bk_$v.json')); n=j['slices']
print('$v', round(j['ms_per_slice'],2), [(r['step'], round(r['ms']/n,3)) for r in j['rows'] if r['step'] in (241, 601, 782, 1605, 1161, 649)])
PY
done
