set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python bench.py > gpurun_out/bench61.json 2> gpurun_out/bench61.err; echo bench rc $?
tail -3 gpurun_out/bench61.err; cat gpurun_out/bench61.json
