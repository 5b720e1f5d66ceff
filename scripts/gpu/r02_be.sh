set -x
timeout 1500 python scripts/ab_compare.py cfg5 8 3 "" "chain_minb=2" 2>&1 | grep -E "median|rror"
STN_DEBUG=sweep_debug,chain_minb=2 timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_be.json > gpurun_out/steps_cfg5_be.txt 2>&1; grep -E "slices|rror" gpurun_out/steps_cfg5_be.txt; python - <<PY
import json
a=json.load(open('gpurun_out/steps_cfg5_bc.json')); b=json.load(open('gpurun_out/steps_cfg5_be.json'))
ra={r['step']:r['ms']/a['slices'] for r in a['rows']}; rb={r['step']:r['ms']/b['slices'] for r in b['rows']}
d=sorted((rb[s]-ra[s], s, round(ra[s],3), round(rb[s],3)) for s in ra if s in rb)
print(d[:12]); print(d[-12:])
PY
