set -x
nproc; free -g | head -2
timeout 1500 python bench.py --impl reference > gpurun_out/ref_cfg5.json 2> gpurun_out/ref_cfg5.err; tail -2 gpurun_out/ref_cfg5.err; cat gpurun_out/ref_cfg5.json | cut -c1-1500
