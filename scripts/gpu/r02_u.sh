set -x
STN_DEBUG=tcf=0 timeout 600 python scripts/gemm_ab.py
STN_DEBUG=tcf=0,gemm_bk=16 timeout 600 python scripts/gemm_ab.py
STN_DEBUG=gemm_bk=16 timeout 600 python scripts/step_profile.py cfg4 fast 4 gpurun_out/steps_cfg4_u16.json > gpurun_out/steps_cfg4_u16.txt 2>&1; head -5 gpurun_out/steps_cfg4_u16.txt
timeout 600 python scripts/step_profile.py cfg4 fast 4 gpurun_out/steps_cfg4_u.json > gpurun_out/steps_cfg4_u.txt 2>&1; head -5 gpurun_out/steps_cfg4_u.txt
python -c "
import sys; sys.path.insert(0,'.')
from paper_2005_06787_b200 import ExecutablePlan
import bench
p=ExecutablePlan.load(bench.plan_file('cfg5'), device=0, mode='fast'); print('cfg5 arena GiB/slice', p.info.arena_bytes_per_slice/2**30)"
