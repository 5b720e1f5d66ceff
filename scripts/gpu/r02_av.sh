set -x
for v in "chain_multi_log=5" ""; do tag=$(echo "x$v" | tr -c 'a-z0-9\n' '_')
STN_DEBUG=sweep_debug,$v timeout 600 python scripts/step_profile.py cfg4 fast 4 gpurun_out/steps_cfg4_av$tag.json > gpurun_out/steps_cfg4_av$tag.txt 2>&1; grep -E "^chain [0-9]|chain kernel|slices|rror" gpurun_out/steps_cfg4_av$tag.txt | head -40; sed -n '/step kernel/,+12p' gpurun_out/steps_cfg4_av$tag.txt
done
