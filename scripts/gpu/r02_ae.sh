set -x
timeout 900 python scripts/ab_compare.py cfg5 4 3 "" "chain_single=1" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg4 8 3 "" "chain_single=1" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 3 "" "chain_single=1" 2>&1 | grep -E "median|rror"
for c in cfg5:2 cfg2:16; do cfg=${c%:*}; n=${c#*:}
STN_DEBUG=sweep_debug,chain_single=1 timeout 600 python scripts/step_profile.py $cfg fast $n gpurun_out/steps_${cfg}_ae.json > gpurun_out/steps_${cfg}_ae.txt 2>&1; grep -E "slices" gpurun_out/steps_${cfg}_ae.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "fused_chains" 2>&1 | tail -2
