mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r75_bench.json 2> gpurun_out/r75_bench.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/r75_bench.json')); print(d['value'], d['e2e'], d['roofline']['frac'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/r75_ref.json 2>&1; echo ref=$?; tail -c 300 gpurun_out/r75_ref.json
