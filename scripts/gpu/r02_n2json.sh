set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/n2_stdout.txt 2> gpurun_out/n2_stderr.txt; echo rc $?
wc -l gpurun_out/n2_stdout.txt; cut -c1-200 gpurun_out/n2_stdout.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > gpurun_out/n2_ref_stdout.txt 2> gpurun_out/n2_ref_stderr.txt; echo rc $?
wc -l gpurun_out/n2_ref_stdout.txt; cut -c1-300 gpurun_out/n2_ref_stdout.txt
