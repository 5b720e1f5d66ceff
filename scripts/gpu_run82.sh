mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r82_bench.json 2> gpurun_out/r82_bench.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/r82_bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'], d['cpu_baseline']['value'])"
