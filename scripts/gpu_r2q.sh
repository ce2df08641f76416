timeout -s KILL 300 python scripts/sanitize_cases.py 2>&1 | tail -12 && \
timeout -s KILL 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -25 gpurun_out/memcheck.log
