mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
STN_PLAN_TIMING=1 timeout 300 python scripts/e2e_breakdown.py 2>&1 | tail -9
