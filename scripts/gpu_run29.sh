rm -rf gpurun_out; mkdir -p gpurun_out
STN_PLAN_DUMP=1 timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/r29_prof.txt 2> gpurun_out/r29_dump.txt; echo prof=$?
head -40 gpurun_out/r29_dump.txt
