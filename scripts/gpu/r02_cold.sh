set -x
export STN_JIT_CACHE=/tmp/cold_jit_cache
rm -rf $STN_JIT_CACHE
timeout 900 python -c "
import time, torch
t=time.time()
import bench
from paper_2005_06787_b200 import ExecutablePlan, build_branch_cache
for c in ['cfg5','cfg4','cfg2']:
    t0=time.time(); p=ExecutablePlan.load(bench.plan_file(c), device=0, mode='fast'); t1=time.time()
    print(c, 'plan create (cold NVRTC)', round(t1-t0,1), 's', p.kernel_mix(), flush=True)
    p.close()
    t0=time.time(); p=ExecutablePlan.load(bench.plan_file(c), device=0, mode='fast'); print(c, 'again (disk cache)', round(time.time()-t0,1), 's', flush=True); p.close()
"
unset STN_JIT_CACHE
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
