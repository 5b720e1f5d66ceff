set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > gpurun_out/n2_ref_stdout.txt 2> gpurun_out/n2_ref_stderr.txt; echo rc $?
wc -l gpurun_out/n2_ref_stdout.txt; cut -c1-400 gpurun_out/n2_ref_stdout.txt
