set -x
for c in cfg5:2 cfg4:4 cfg2:16; do cfg=${c%:*}; n=${c#*:}
STN_DEBUG=sweep_debug,chain_single=2,chain_min_bits=20 timeout 600 python scripts/step_profile.py $cfg fast $n gpurun_out/steps_${cfg}_z.json > gpurun_out/steps_${cfg}_z.txt 2>&1; grep -E "^chain [0-9]|slices" gpurun_out/steps_${cfg}_z.txt | head -80
STN_DEBUG=sweep_debug,chain_min_bits=20 timeout 600 python scripts/step_profile.py $cfg fast $n gpurun_out/steps_${cfg}_z0.json > gpurun_out/steps_${cfg}_z0.txt 2>&1; grep -E "slices" gpurun_out/steps_${cfg}_z0.txt | head -80
done
