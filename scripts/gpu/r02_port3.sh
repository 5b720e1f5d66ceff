set -x
CFG5_SLICES=11400714819323198485 timeout 1500 python scripts/cfg5_parity.py 2>&1 | tail -4
ls -la gpurun_out/cfg5_oracle_*.npy
