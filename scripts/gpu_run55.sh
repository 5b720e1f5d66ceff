rm -rf gpurun_out; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/r55_bench.log 2>&1; echo bench=$?
grep "^{" gpurun_out/r55_bench.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['traffic'], d['roofline']['algorithmic_bytes_per_launch'])"
