set -x
for v in "perm_tb=11" "perm_tb=12" "perm_tb=13" "perm_tb=10"; do STN_DEBUG=$v timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_bb_$v.json > gpurun_out/steps_cfg5_bb_$v.txt 2>&1; python - <<PY
import json
j=json.load(open('gpurun_out/steps_cfg5_bb_$v.json')); n=j['slices']
print('$v', round(j['ms_per_slice'],2), [(r['step'], round(r['ms']/n,3)) for r in j['rows'] if r['step'] in (259, 816, 1306, 1394)])
PY
done
timeout 900 python bench.py > gpurun_out/bench_cfg5_bb.json 2> gpurun_out/bench_cfg5_bb.err; python -c "
import json; j=json.load(open('gpurun_out/bench_cfg5_bb.json')); r=j['roofline']; print('cfg5', j['value'], j['ms_per_step'], j['e2e']['value'], r['kernel'], round(r['frac'],3), j['clocks'])"
