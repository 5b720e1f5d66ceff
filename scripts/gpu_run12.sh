set -x
nvidia-smi --query-gpu=index,name --format=csv
timeout 1800 python -m pytest tests -m gpu -q -s --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/step_profile_cfg2_default.txt 2>&1; echo prof=$?
timeout 900 python scripts/run_cfg5.py 2 > gpurun_out/cfg5.log 2>&1; echo cfg5=$?
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 --cpu-baseline 0 > gpurun_out/bench_cfg2_n1.log 2>&1; echo bench1=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_cfg2_n2.log 2>&1; echo bench2=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 --ref-budget 5 > gpurun_out/bench_ref_n2.log 2>&1; echo benchref=$?
grep -E "FAIL|passed|failed" gpurun_out/pytest_gpu.log | tail -5; head -24 gpurun_out/step_profile_cfg2_default.txt; head -12 gpurun_out/cfg5.log; tail -c 400 gpurun_out/bench_cfg2_n1.log; tail -c 1200 gpurun_out/bench_cfg2_n2.log; tail -c 600 gpurun_out/bench_ref_n2.log
