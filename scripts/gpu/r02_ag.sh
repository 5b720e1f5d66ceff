set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_chains or cfg2 or cfg1" 2>&1 | tail -2
timeout 900 python scripts/ab_compare.py cfg5 4 3 "chain_vec=1" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg4 8 3 "chain_vec=1" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 3 "chain_vec=1" "" 2>&1 | grep -E "median|rror"
for c in cfg5:2 cfg2:16; do cfg=${c%:*}; n=${c#*:}
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py $cfg fast $n gpurun_out/steps_${cfg}_ag.json > gpurun_out/steps_${cfg}_ag.txt 2>&1; grep -E "slices" gpurun_out/steps_${cfg}_ag.txt
done
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
