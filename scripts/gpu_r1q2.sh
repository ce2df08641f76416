timeout -s KILL 600 python -m pytest tests/test_gpu_depthwise.py -x -q 2>&1 | grep -E "Error|error|assert|^E " | head -20
CO_LIB_VARIANT=px3 timeout -s KILL 300 python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -3
