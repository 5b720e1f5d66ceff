mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python scripts/step_profile.py cfg2 > gpurun_out/r63_prof.txt 2>&1; echo prof=$?; head -30 gpurun_out/r63_prof.txt
timeout 900 python bench.py --cpu-baseline 0 > gpurun_out/bench63.json 2> gpurun_out/bench63.err; echo bench rc $?
python -c "import json; d=json.load(open('gpurun_out/bench63.json')); print(d['value'], d['e2e'], d['roofline']['frac'])"
