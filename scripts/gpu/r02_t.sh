set -x
timeout 600 python scripts/sanitize_target.py > gpurun_out/san_plain.log 2>&1 && timeout 2400 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python scripts/sanitize_target.py > gpurun_out/san_memcheck.log 2>&1; tail -15 gpurun_out/san_memcheck.log
