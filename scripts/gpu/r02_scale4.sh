set -x
nvidia-smi --query-gpu=index,name --format=csv,noheader
export CUDA_VISIBLE_DEVICES=0
timeout 900 python bench.py > gpurun_out/sc_cfg5_n1.json 2> gpurun_out/sc_cfg5_n1.err
unset CUDA_VISIBLE_DEVICES
for N in 2 4; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N > gpurun_out/sc_cfg5_n$N.json 2> gpurun_out/sc_cfg5_n$N.err; done
for N in 1 2 4; do python -c "
import json; j=json.load(open('gpurun_out/sc_cfg5_n$N.json')); print($N, j['value'], j['ms_per_step'], j['e2e']['value'], j['clocks'])"; done
timeout 600 python scripts/multi_abi_bench.py > gpurun_out/multi_abi_n4.txt 2>&1; cat gpurun_out/multi_abi_n4.txt
