set -x
STN_DEBUG=plan_dump timeout 600 python scripts/step_profile.py cfg5 fast 1 > gpurun_out/dump_cfg5.txt 2>&1; grep -c "^step " gpurun_out/dump_cfg5.txt
for c in cfg5:2 cfg4:4 cfg2:16; do cfg=${c%:*}; n=${c#*:}
for v in "chain_single=1" "chain_single=1,chain_pf_log=4"; do tag=$(echo $v | tr -c 'a-z0-9\n' '_')
STN_DEBUG=sweep_debug,$v timeout 600 python scripts/step_profile.py $cfg fast $n gpurun_out/steps_${cfg}_aa_$tag.json > gpurun_out/steps_${cfg}_aa_$tag.txt 2>&1; grep -E "slices" gpurun_out/steps_${cfg}_aa_$tag.txt
done; done
STN_DEBUG=chain_single=1 timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
