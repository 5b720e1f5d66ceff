set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_chains" 2>&1 | tail -3
for c in cfg5:2 cfg2:16; do cfg=${c%:*}; n=${c#*:}
for v in "chain_single=1"; do tag=$(echo $v | tr -c 'a-z0-9\n' '_')
STN_DEBUG=sweep_debug,$v timeout 600 python scripts/step_profile.py $cfg fast $n gpurun_out/steps_${cfg}_ab_$tag.json > gpurun_out/steps_${cfg}_ab_$tag.txt 2>&1; grep -E "slices|rror" gpurun_out/steps_${cfg}_ab_$tag.txt
done; done
STN_DEBUG=chain_single=1 timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
