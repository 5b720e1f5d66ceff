rm -rf gpurun_out; mkdir -p gpurun_out
timeout 300 python scripts/step_profile.py cfg2 > gpurun_out/r47_prof.txt 2>&1; head -60 gpurun_out/r47_prof.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/r47_bench.log 2>&1; echo bench=$?
grep "^{" gpurun_out/r47_bench.log | cut -c1-400
