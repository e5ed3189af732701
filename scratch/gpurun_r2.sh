mkdir -p gpurun_out
python scripts/sanitize_small.py > gpurun_out/r2j_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python scripts/sanitize_small.py > gpurun_out/r2j_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_memcheck.log
