timeout -s KILL 120 python -m pytest tests/test_gpu_dense_tc.py -x -q -k "cta_pair" 2>&1 | tail -15
