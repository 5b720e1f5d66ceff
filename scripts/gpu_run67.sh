mkdir -p gpurun_out
nvidia-smi -L
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --cpu-baseline 0 > gpurun_out/r67_bench_n$n.json 2> gpurun_out/r67_bench_n$n.err; echo n=$n rc=$?
python -c "import json; d=json.loads(open('gpurun_out/r67_bench_n$n.json').read().strip().splitlines()[-1]); print($n, d['value'], d['e2e']['value'], d['ms_per_step'])"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 4 --steps 1 --warmup 0 > gpurun_out/r67_ref_n4.json 2>&1; echo ref rc=$?; tail -c 600 gpurun_out/r67_ref_n4.json
