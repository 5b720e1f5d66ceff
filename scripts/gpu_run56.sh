rm -rf gpurun_out; mkdir -p gpurun_out
for c in cfg3 cfg4; do timeout 600 python scripts/step_profile.py $c > gpurun_out/r56_prof_$c.txt 2>&1; echo $c=$?; head -4 gpurun_out/r56_prof_$c.txt; done
timeout 900 python scripts/run_cfg5.py 2 > gpurun_out/r56_cfg5.txt 2>&1; echo cfg5=$?; head -30 gpurun_out/r56_cfg5.txt | cut -c1-400
