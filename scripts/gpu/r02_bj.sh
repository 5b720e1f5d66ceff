set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -2
STN_DEBUG=tcf=2 timeout 300 python scripts/gemm_ab.py 2>&1 | tail -4
for c in cfg5:2 cfg4:4; do cfg=${c%:*}; n=${c#*:}
timeout 600 python scripts/step_profile.py $cfg fast $n gpurun_out/steps_${cfg}_bj.json > gpurun_out/steps_${cfg}_bj.txt 2>&1; grep -E "slices|rror" gpurun_out/steps_${cfg}_bj.txt; python - <<PY
import json
j=json.load(open('gpurun_out/steps_${cfg}_bj.json')); n=j['slices']
print([(r['step'], r['kernel'], round(r['ms']/n,3)) for r in j['rows'] if r['kernel']=='gemm_tc'][:8])
PY
done
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
