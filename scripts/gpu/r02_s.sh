set -x
nvidia-smi --query-gpu=index,name --format=csv,noheader
N=$(nvidia-smi --query-gpu=index --format=csv,noheader | wc -l)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --config cfg5 > gpurun_out/bench_cfg5_n$N.json 2> gpurun_out/bench_cfg5_n$N.err; grep -v Warning gpurun_out/bench_cfg5_n$N.err | tail -2; cut -c1-250 gpurun_out/bench_cfg5_n$N.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --config cfg5 > gpurun_out/bench_cfg5_n2.json 2> gpurun_out/bench_cfg5_n2.err; cut -c1-250 gpurun_out/bench_cfg5_n2.json
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_dropin.py -x -q 2>&1 | tail -2
timeout 600 python scripts/multi_abi_bench.py > gpurun_out/multi_abi_n$N.txt 2>&1; cat gpurun_out/multi_abi_n$N.txt | cut -c1-200
