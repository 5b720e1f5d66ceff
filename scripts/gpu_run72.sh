rm -rf gpurun_out; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/r72_bench.json 2> gpurun_out/r72_bench.err; echo bench=$?
timeout 300 python scripts/step_profile.py cfg2 > gpurun_out/r72_prof.txt 2>&1; echo prof=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r72_launches.csv python scripts/ncu_target.py cfg2 1 > gpurun_out/r72_l.log 2>&1; echo ncu=$?
timeout 900 ncu --kernel-name-base demangled --set full --import-source on --clock-control none -k 'regex:k_absorb_direct<\(bool\)0, \(int\)16, \(int\)8, \(bool\)1>' -s 2 -c 1 -o gpurun_out/r72_direct python scripts/ncu_target.py cfg2 1 > gpurun_out/r72_ncu1.log 2>&1; echo ncu1=$?
timeout 900 ncu --kernel-name-base demangled --set full --import-source on --clock-control none -k 'regex:k_splitk_partial' -c 1 -o gpurun_out/r72_splitk python scripts/ncu_target.py cfg2 1 > gpurun_out/r72_ncu2.log 2>&1; echo ncu2=$?
python -c "import json; d=json.load(open('gpurun_out/r72_bench.json')); print(d['value'], d['e2e'], d['roofline']['frac'], d['clocks'])"
