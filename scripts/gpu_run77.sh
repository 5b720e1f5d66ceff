mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
for c in cfg3 cfg4; do timeout 600 python scripts/step_profile.py $c > gpurun_out/r77_prof_$c.txt 2>&1; echo $c=$?; sed -n 2,6p gpurun_out/r77_prof_$c.txt; done
timeout 900 python bench.py --cpu-baseline 0 > gpurun_out/r77_bench.json 2> gpurun_out/r77_bench.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/r77_bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
