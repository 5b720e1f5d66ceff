set -x
for c in cfg5:2 cfg4:4 cfg2:16; do cfg=${c%:*}; n=${c#*:}
STN_DEBUG=sweep_debug,chain_single=1 timeout 600 python scripts/step_profile.py $cfg fast $n gpurun_out/steps_${cfg}_y.json > gpurun_out/steps_${cfg}_y.txt 2>&1; grep -E "^chain [0-9]|slices" gpurun_out/steps_${cfg}_y.txt | head -60
done
STN_DEBUG=chain_single=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg1 or cfg2 or rt_" 2>&1 | tail -3
